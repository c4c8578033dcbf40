"""The small parity meshes run one SELL slice per warp at the default grid
size: the grid-stride multi-slice loops and the
next-slice prefetch of every gather / Krylov / AMG kernel were then only
compared with the oracle at 50M cells.  Here the operator, solver and PISO
parity suites are re-run in a fresh process with DFVM_MAX_BLOCKS caps (read
once at library load), so every warp walks several slices and every
grid-stride loop wraps, against the same oracle tolerances."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

SEL = ("test_gpu_parity.py::test_grad_scalar_and_vector test_gpu_parity.py::test_div "
       "test_gpu_parity.py::test_laplacian test_gpu_parity.py::test_grad_from_face_values "
       "test_gpu_parity.py::test_interpolate test_gpu_piso.py::test_momentum_assembly_and_apply "
       "test_gpu_piso.py::test_pressure_solve test_gpu_piso.py::test_cavity_steps "
       "test_gpu_piso.py::test_pipe_nonorth_steps test_gpu_piso.py::test_htree_windkessel_outlets "
       "test_gpu_piso.py::test_c3_cylinder_poly_piso test_gpu_adjoint.py").split()


@pytest.mark.parametrize("cap", ["1", "3"])
def test_parity_suites_with_capped_grids(cap):
    env = dict(os.environ, DFVM_MAX_BLOCKS=cap)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider"] +
                       [os.path.join(HERE, s) for s in SEL], cwd=os.path.dirname(HERE), env=env,
                       capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
