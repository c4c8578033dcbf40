# Build all native code in-tree (the .so files travel to the GPU box with gpurun).
#   synth/libsynth.so                      seeded input generators (test/bench tooling)
#   oracle/liboracle.so                    CPU fp64 oracle (test infrastructure only)
#   paper_2603_15920_b200/libdfvm.so       the product: host pipeline + sm_100a kernels, C ABI
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
CXXFLAGS  := -O2 -std=c++17 -fPIC -Wall -Wno-unused-function
ORACLE_FLAGS := -O2 -std=c++17 -fPIC -fno-fast-math -ffp-contract=off
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fopenmp \
             --expt-relaxed-constexpr -Iinclude -Xptxas -v
PKG       := paper_2603_15920_b200
CSRC      := $(PKG)/csrc
HOST_SRC  := $(wildcard $(CSRC)/*.cpp)
DEV_SRC   := $(wildcard $(CSRC)/*.cu)
HDRS      := $(wildcard $(CSRC)/*.h $(CSRC)/*.cuh) include/dfvm.h
HOST_OBJ  := $(patsubst $(CSRC)/%.cpp,build/%.o,$(HOST_SRC))
DEV_OBJ   := $(patsubst $(CSRC)/%.cu,build/%.cu.o,$(DEV_SRC))
NCCL_INC  ?= $(shell python -c "import nvidia.nccl,os;print(os.path.join(nvidia.nccl.__path__[0],'include'))" 2>/dev/null)
NCCL_LIB  ?= $(shell python -c "import nvidia.nccl,os;print(os.path.join(nvidia.nccl.__path__[0],'lib'))" 2>/dev/null)

all: synth/libsynth.so oracle/liboracle.so $(if $(DEV_SRC),$(PKG)/libdfvm.so)

synth/libsynth.so: synth/meshgen.cpp
	$(CXX) $(CXXFLAGS) -O3 -shared -o $@ $<

oracle/liboracle.so: $(wildcard oracle/*.cpp oracle/*.h)
	$(CXX) $(ORACLE_FLAGS) -shared -o $@ $(wildcard oracle/*.cpp)

build/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -O3 -fopenmp -Iinclude -I/usr/local/cuda/include -c -o $@ $<

build/%.cu.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(PKG)/libdfvm.so: $(HOST_OBJ) $(DEV_OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fopenmp -lcudart -ldl

clean:
	rm -rf build synth/libsynth.so oracle/liboracle.so $(PKG)/libdfvm.so

.PHONY: all clean
