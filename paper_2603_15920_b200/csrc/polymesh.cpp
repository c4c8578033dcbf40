// polymesh.cpp — OpenFOAM ASCII polyMesh reader (SURVEY.md §8(f) NEXT-4
// "OpenFOAM ASCII case reader"; "reads OpenFOAM polyMesh
// files directly", Table 1 P:394 "OpenFOAM drop-in").
//
// Reads <dir>/{points, faces, owner, neighbour, boundary} (dir = a case
// directory, its constant/polyMesh, or the polyMesh directory itself) into
// the arrays dfvm_mesh_create takes.  ASCII format only (FoamFile header
// `format ascii`); `binary` and compressed files are rejected with
// DFVM_E_INVALID_ARG naming the file.  Host only; no device work.
#include <algorithm>
#include <cctype>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "internal.h"

struct dfvm_polymesh {
  std::vector<double> points;
  std::vector<int64_t> face_offsets;
  std::vector<int32_t> face_points, owner, neighbour;
  std::vector<std::string> names;
  std::vector<dfvm_patch_desc> patches;
  int64_t n_cells = 0;
};

namespace dfvm {
namespace {

// Tokeniser over one file: words, numbers and the punctuation ( ) { } ; with
// C/C++ comments removed.
struct Lexer {
  std::string s, file;
  size_t i = 0;
  bool ok = true;
  std::string err;

  void fail(const std::string& m) {
    if (ok) err = file + ": " + m;
    ok = false;
  }
  void skip_ws() {
    for (;;) {
      while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
      if (i + 1 < s.size() && s[i] == '/' && s[i + 1] == '/') {
        while (i < s.size() && s[i] != '\n') ++i;
      } else if (i + 1 < s.size() && s[i] == '/' && s[i + 1] == '*') {
        const size_t e = s.find("*/", i + 2);
        i = e == std::string::npos ? s.size() : e + 2;
      } else {
        return;
      }
    }
  }
  // next token ("" at end of file)
  std::string next() {
    skip_ws();
    if (i >= s.size()) return "";
    const char c = s[i];
    if (std::strchr("(){};", c)) { ++i; return std::string(1, c); }
    if (c == '"') {
      const size_t e = s.find('"', i + 1);
      std::string t = s.substr(i + 1, (e == std::string::npos ? s.size() : e) - i - 1);
      i = e == std::string::npos ? s.size() : e + 1;
      return t;
    }
    const size_t b = i;
    while (i < s.size() && !std::isspace((unsigned char)s[i]) && !std::strchr("(){};", s[i])) ++i;
    return s.substr(b, i - b);
  }
  std::string peek() { const size_t k = i; std::string t = next(); i = k; return t; }
  void expect(const char* t) {
    const std::string g = next();
    if (g != t) fail(std::string("expected '") + t + "', found '" + g + "'");
  }
  int64_t integer() {
    const std::string t = next();
    char* e = nullptr;
    const long long v = std::strtoll(t.c_str(), &e, 10);
    if (t.empty() || *e) { fail("expected an integer, found '" + t + "'"); return 0; }
    return v;
  }
  double real() {
    const std::string t = next();
    char* e = nullptr;
    const double v = std::strtod(t.c_str(), &e);
    if (t.empty() || *e) { fail("expected a number, found '" + t + "'"); return 0; }
    return v;
  }
  // skip a { ... } dictionary (nested)
  void skip_dict() {
    expect("{");
    int depth = 1;
    while (ok && depth > 0) {
      const std::string t = next();
      if (t.empty()) { fail("unterminated dictionary"); return; }
      if (t == "{") ++depth;
      else if (t == "}") --depth;
    }
  }
  // FoamFile header: require format ascii; leaves the lexer after the header
  void header() {
    if (peek() != "FoamFile") return;   // headerless files are accepted
    next();
    expect("{");
    while (ok) {
      const std::string k = next();
      if (k == "}") return;
      if (k.empty()) { fail("unterminated FoamFile header"); return; }
      std::string v;
      for (std::string t = next(); ok && t != ";"; t = next()) {
        if (t.empty()) { fail("unterminated header entry"); return; }
        v += t;
      }
      if (k == "format" && v != "ascii") fail("format '" + v + "' is not supported (ASCII polyMesh only)");
    }
  }
};

bool load(const std::string& path, Lexer& L) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  L.s = ss.str();
  L.file = path;
  if (L.s.size() >= 2 && (unsigned char)L.s[0] == 0x1f && (unsigned char)L.s[1] == 0x8b)
    L.fail("gzip-compressed file (decompress it first)");
  return true;
}

// "N ( ... )" list of labels
void label_list(Lexer& L, std::vector<int32_t>& out) {
  const int64_t n = L.integer();
  if (!L.ok) return;
  if (n < 0 || n >= (int64_t)1 << 31) { L.fail("list size out of range"); return; }
  out.resize((size_t)n);
  L.expect("(");
  for (int64_t k = 0; k < n && L.ok; ++k) {
    const int64_t v = L.integer();
    if (v < INT32_MIN || v > INT32_MAX) L.fail("label out of int32 range");
    out[(size_t)k] = (int32_t)v;
  }
  L.expect(")");
}

bool find_dir(const std::string& dir, std::string& out) {
  for (const char* sub : {"/constant/polyMesh", "/polyMesh", ""}) {
    const std::string d = dir + sub;
    std::ifstream f(d + "/points");
    if (f) { out = d; return true; }
  }
  return false;
}

}  // namespace
}  // namespace dfvm

using namespace dfvm;

extern "C" {

dfvm_status dfvm_polymesh_read(const char* dir, dfvm_polymesh** out) {
  set_error(DFVM_OK, "", -1);
  if (!dir || !out) { set_error(DFVM_E_INVALID_ARG, "NULL argument"); return DFVM_E_INVALID_ARG; }
  std::string d;
  if (!find_dir(dir, d)) {
    set_error(DFVM_E_INVALID_ARG, std::string("no polyMesh/points under '") + dir + "'");
    return DFVM_E_INVALID_ARG;
  }
  std::unique_ptr<dfvm_polymesh> M(new dfvm_polymesh());
  auto bad = [&](const Lexer& L) {
    set_error(DFVM_E_INVALID_ARG, L.err);
    return DFVM_E_INVALID_ARG;
  };
  // points: N ( (x y z) ... )
  {
    Lexer L;
    if (!load(d + "/points", L)) { set_error(DFVM_E_INVALID_ARG, "cannot read " + d + "/points"); return DFVM_E_INVALID_ARG; }
    L.header();
    const int64_t n = L.integer();
    if (L.ok && (n < 0 || n >= (int64_t)1 << 31)) L.fail("point count out of range");
    L.expect("(");
    M->points.resize(L.ok ? (size_t)(3 * n) : 0);
    for (int64_t k = 0; k < n && L.ok; ++k) {
      L.expect("(");
      for (int c = 0; c < 3; ++c) M->points[(size_t)(3 * k + c)] = L.real();
      L.expect(")");
    }
    L.expect(")");
    if (!L.ok) return bad(L);
  }
  // faces: N ( k(a b c ...) ... )
  {
    Lexer L;
    if (!load(d + "/faces", L)) { set_error(DFVM_E_INVALID_ARG, "cannot read " + d + "/faces"); return DFVM_E_INVALID_ARG; }
    L.header();
    const int64_t n = L.integer();
    if (L.ok && (n < 0 || n >= (int64_t)1 << 31)) L.fail("face count out of range");
    L.expect("(");
    M->face_offsets.assign(1, 0);
    for (int64_t k = 0; k < n && L.ok; ++k) {
      const int64_t m = L.integer();
      if (L.ok && m < 3) L.fail("face " + std::to_string(k) + " has fewer than 3 points");
      L.expect("(");
      for (int64_t j = 0; j < m && L.ok; ++j) M->face_points.push_back((int32_t)L.integer());
      L.expect(")");
      M->face_offsets.push_back((int64_t)M->face_points.size());
    }
    L.expect(")");
    if (!L.ok) return bad(L);
  }
  for (const char* nm : {"owner", "neighbour"}) {
    Lexer L;
    if (!load(d + "/" + nm, L)) { set_error(DFVM_E_INVALID_ARG, "cannot read " + d + "/" + nm); return DFVM_E_INVALID_ARG; }
    L.header();
    label_list(L, nm[0] == 'o' ? M->owner : M->neighbour);
    if (!L.ok) return bad(L);
  }
  // boundary: N ( name { type t; nFaces n; startFace s; ... } ... )
  {
    Lexer L;
    if (!load(d + "/boundary", L)) { set_error(DFVM_E_INVALID_ARG, "cannot read " + d + "/boundary"); return DFVM_E_INVALID_ARG; }
    L.header();
    const int64_t n = L.integer();
    L.expect("(");
    for (int64_t k = 0; k < n && L.ok; ++k) {
      const std::string name = L.next();
      L.expect("{");
      std::string type;
      int64_t nf = -1, sf = -1;
      while (L.ok) {
        const std::string key = L.next();
        if (key == "}") break;
        if (key.empty()) { L.fail("unterminated patch dictionary"); break; }
        if (L.peek() == "{") { L.skip_dict(); continue; }
        std::vector<std::string> val;
        int depth = 0;
        for (std::string t = L.next(); L.ok && (t != ";" || depth > 0); t = L.next()) {
          if (t.empty()) { L.fail("unterminated entry '" + key + "'"); break; }
          if (t == "(") ++depth;
          if (t == ")") --depth;
          val.push_back(t);
        }
        if (key == "type" && val.size() == 1) type = val[0];
        else if (key == "nFaces" && val.size() == 1) nf = std::atoll(val[0].c_str());
        else if (key == "startFace" && val.size() == 1) sf = std::atoll(val[0].c_str());
      }
      if (!L.ok) break;
      if (nf < 0 || sf < 0) { L.fail("patch '" + name + "' lacks nFaces / startFace"); break; }
      int32_t kind = DFVM_PATCH_GENERIC;
      if (type == "wall") kind = DFVM_PATCH_WALL;
      else if (type == "empty") kind = DFVM_PATCH_EMPTY;
      else if (type == "cyclic" || type == "cyclicAMI" || type == "processor" || type == "wedge") {
        L.fail("patch '" + name + "' of type '" + type + "' is not supported");
        break;
      }
      M->names.push_back(name);
      M->patches.push_back(dfvm_patch_desc{nullptr, (dfvm_patch_kind)kind, sf, nf});
    }
    L.expect(")");
    if (!L.ok) return bad(L);
  }
  for (size_t k = 0; k < M->patches.size(); ++k) M->patches[k].name = M->names[k].c_str();
  const int64_t nf = (int64_t)M->face_offsets.size() - 1;
  if ((int64_t)M->owner.size() != nf || (int64_t)M->neighbour.size() > nf) {
    set_error(DFVM_E_MESH_CONSISTENCY, "owner / neighbour sizes do not match the face count");
    return DFVM_E_MESH_CONSISTENCY;
  }
  int64_t nc = 0;
  for (int32_t v : M->owner) nc = std::max<int64_t>(nc, (int64_t)v + 1);
  for (int32_t v : M->neighbour) nc = std::max<int64_t>(nc, (int64_t)v + 1);
  M->n_cells = nc;
  *out = M.release();
  return DFVM_OK;
}

dfvm_status dfvm_polymesh_sizes(const dfvm_polymesh* m, int64_t* n_points, int64_t* n_faces,
                                int64_t* n_face_points, int64_t* n_internal, int32_t* n_patches, int64_t* n_cells) {
  if (!m) { set_error(DFVM_E_INVALID_ARG, "NULL argument"); return DFVM_E_INVALID_ARG; }
  if (n_points) *n_points = (int64_t)m->points.size() / 3;
  if (n_faces) *n_faces = (int64_t)m->face_offsets.size() - 1;
  if (n_face_points) *n_face_points = (int64_t)m->face_points.size();
  if (n_internal) *n_internal = (int64_t)m->neighbour.size();
  if (n_patches) *n_patches = (int32_t)m->patches.size();
  if (n_cells) *n_cells = m->n_cells;
  return DFVM_OK;
}

dfvm_status dfvm_polymesh_arrays(const dfvm_polymesh* m, const double** points, const int64_t** face_offsets,
                                 const int32_t** face_points, const int32_t** owner, const int32_t** neighbour,
                                 const dfvm_patch_desc** patches) {
  if (!m) { set_error(DFVM_E_INVALID_ARG, "NULL argument"); return DFVM_E_INVALID_ARG; }
  if (points) *points = m->points.data();
  if (face_offsets) *face_offsets = m->face_offsets.data();
  if (face_points) *face_points = m->face_points.data();
  if (owner) *owner = m->owner.data();
  if (neighbour) *neighbour = m->neighbour.data();
  if (patches) *patches = m->patches.data();
  return DFVM_OK;
}

dfvm_status dfvm_polymesh_destroy(dfvm_polymesh* m) {
  delete m;
  return DFVM_OK;
}

}  // extern "C"
