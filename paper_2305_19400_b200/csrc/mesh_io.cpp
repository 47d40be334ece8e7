// mesh_io.cpp -- host-side mesh import and partitioning for the unstructured
// path.
//
//   bte_mesh_read   Gmsh (ASCII 2.2 and 4.1) and MEDIT (.mesh, ASCII) files ->
//                   vertex / cell arrays for bte_create_umesh.  P:L544-547: "A
//                   mesh must either be imported from a Gmsh or MEDIT
//                   formatted mesh file, or generated internally".
//   bte_partition_rcb
//                   recursive coordinate bisection of the cell centroids: a
//                   cell order whose contiguous ranges [r N/P, (r+1) N/P) are
//                   compact parts, for meshes given in any order (the paper
//                   partitions with Metis; SPEC partitions cells by
//                   recursive bisection).  bte_create_umesh's cell-range
//                   partition then follows these parts.
//
// No CUDA here: both are host-only and callable without a GPU.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/bte.h"

namespace {

thread_local std::string g_mesh_err;

bte_status mfail(const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_mesh_err = buf;
  return BTE_EINVAL;
}

struct Raw {
  int dim = 0;
  std::vector<double> verts;          // [n][3]
  std::vector<int64_t> tri, quad, tet, hex;  // 0-based vertex indices
};

// Reads whitespace-separated tokens line by line (comments '#' in MEDIT).
struct Tok {
  std::istream &in;
  std::string line;
  std::istringstream ls;
  bool medit;
  explicit Tok(std::istream &s, bool m) : in(s), medit(m) {}
  bool next(std::string &t) {
    while (!(ls >> t)) {
      if (!std::getline(in, line)) return false;
      if (medit) {
        const size_t h = line.find('#');
        if (h != std::string::npos) line.resize(h);
      }
      ls.clear();
      ls.str(line);
    }
    return true;
  }
  bool num(double &x) {
    std::string t;
    if (!next(t)) return false;
    char *end = nullptr;
    x = std::strtod(t.c_str(), &end);
    return end && *end == '\0';
  }
  bool integer(int64_t &x) {
    std::string t;
    if (!next(t)) return false;
    char *end = nullptr;
    x = std::strtoll(t.c_str(), &end, 10);
    return end && *end == '\0';
  }
  // rest of the current line (Gmsh element records have a variable length)
  void drop_line() {
    ls.clear();
    ls.str("");
  }
};

// ---- Gmsh ASCII 2.2: $Nodes n / id x y z; $Elements n / id type ntags tags... nodes
// ---- Gmsh ASCII 4.1: $Nodes nblocks nnodes min max / per block: dim tag param n,
//      n tags, n coordinate triples; $Elements nblocks nelem min max / per block:
//      dim tag type n, then n lines "id nodes..."
// element types: 1 line(2), 2 triangle(3), 3 quadrangle(4), 4 tetrahedron(4),
// 5 hexahedron(8), 6 prism(6), 7 pyramid(5), 15 point(1)
int gmsh_nodes(int type) {
  switch (type) {
    case 1: return 2;
    case 2: return 3;
    case 3: return 4;
    case 4: return 4;
    case 5: return 8;
    case 6: return 6;
    case 7: return 5;
    case 15: return 1;
    default: return -1;
  }
}

bte_status add_elem(Raw &r, int type, const std::vector<int64_t> &nodes) {
  std::vector<int64_t> *dst = type == 2 ? &r.tri : type == 3 ? &r.quad : type == 4 ? &r.tet
                            : type == 5 ? &r.hex : nullptr;
  if (type == 6 || type == 7)
    return mfail("element type %d (prism / pyramid) is not supported: tetrahedra, hexahedra, triangles and "
                 "quadrilaterals only", type);
  if (!dst) return BTE_OK;  // points and lines: boundary tags, not cells
  dst->insert(dst->end(), nodes.begin(), nodes.end());
  return BTE_OK;
}

bte_status read_gmsh(std::istream &in, Raw &r) {
  Tok tk(in, false);
  std::string t;
  double version = 0;
  std::map<int64_t, int64_t> id2idx;  // node tag -> 0-based position
  bool have_nodes = false, have_elems = false;
  while (tk.next(t)) {
    if (t == "$MeshFormat") {
      int64_t ftype, dsize;
      if (!tk.num(version) || !tk.integer(ftype) || !tk.integer(dsize))
        return mfail("bad $MeshFormat section");
      if (ftype != 0) return mfail("binary Gmsh files are not supported (ASCII only)");
      if (!(version >= 2.0 && version < 3.0) && !(version >= 4.0 && version < 5.0))
        return mfail("Gmsh format version %g not supported (2.x or 4.x)", version);
      tk.next(t);  // $EndMeshFormat
    } else if (t == "$Nodes") {
      if (version == 0) return mfail("$Nodes before $MeshFormat");
      if (version < 3.0) {
        int64_t n;
        if (!tk.integer(n) || n < 0) return mfail("bad $Nodes count");
        r.verts.resize(3 * n);
        for (int64_t k = 0; k < n; ++k) {
          int64_t id;
          double x, y, z;
          if (!tk.integer(id) || !tk.num(x) || !tk.num(y) || !tk.num(z)) return mfail("bad node record %lld", (long long)k);
          id2idx[id] = k;
          r.verts[3 * k] = x;
          r.verts[3 * k + 1] = y;
          r.verts[3 * k + 2] = z;
        }
      } else {
        int64_t nb, nn, mn, mx;
        if (!tk.integer(nb) || !tk.integer(nn) || !tk.integer(mn) || !tk.integer(mx)) return mfail("bad $Nodes header");
        r.verts.resize(3 * nn);
        int64_t k = 0;
        for (int64_t bl = 0; bl < nb; ++bl) {
          int64_t edim, etag, param, n;
          if (!tk.integer(edim) || !tk.integer(etag) || !tk.integer(param) || !tk.integer(n))
            return mfail("bad node block header");
          if (param != 0) return mfail("parametric node blocks are not supported");
          std::vector<int64_t> tags(n);
          for (auto &g : tags)
            if (!tk.integer(g)) return mfail("bad node tag");
          for (int64_t q = 0; q < n; ++q, ++k) {
            if (k >= nn) return mfail("more nodes than announced");
            double x, y, z;
            if (!tk.num(x) || !tk.num(y) || !tk.num(z)) return mfail("bad node coordinates");
            id2idx[tags[q]] = k;
            r.verts[3 * k] = x;
            r.verts[3 * k + 1] = y;
            r.verts[3 * k + 2] = z;
          }
        }
        if (k != nn) return mfail("node blocks hold %lld nodes, header says %lld", (long long)k, (long long)nn);
      }
      tk.next(t);  // $EndNodes
      have_nodes = true;
    } else if (t == "$Elements") {
      if (!have_nodes) return mfail("$Elements before $Nodes");
      auto node_index = [&](int64_t id, int64_t *out) -> bool {
        auto it = id2idx.find(id);
        if (it == id2idx.end()) return false;
        *out = it->second;
        return true;
      };
      if (version < 3.0) {
        int64_t n;
        if (!tk.integer(n) || n < 0) return mfail("bad $Elements count");
        for (int64_t k = 0; k < n; ++k) {
          int64_t id, type, ntags;
          if (!tk.integer(id) || !tk.integer(type) || !tk.integer(ntags)) return mfail("bad element record");
          const int nn = gmsh_nodes((int)type);
          if (nn < 0) return mfail("unknown Gmsh element type %lld", (long long)type);
          for (int64_t q = 0; q < ntags; ++q) {
            int64_t tag;
            if (!tk.integer(tag)) return mfail("bad element tags");
          }
          std::vector<int64_t> nodes(nn);
          for (int q = 0; q < nn; ++q) {
            int64_t nid;
            if (!tk.integer(nid) || !node_index(nid, &nodes[q])) return mfail("element %lld: unknown node", (long long)id);
          }
          if (bte_status st = add_elem(r, (int)type, nodes)) return st;
        }
      } else {
        int64_t nb, ne, mn, mx;
        if (!tk.integer(nb) || !tk.integer(ne) || !tk.integer(mn) || !tk.integer(mx)) return mfail("bad $Elements header");
        for (int64_t bl = 0; bl < nb; ++bl) {
          int64_t edim, etag, type, n;
          if (!tk.integer(edim) || !tk.integer(etag) || !tk.integer(type) || !tk.integer(n))
            return mfail("bad element block header");
          const int nn = gmsh_nodes((int)type);
          if (nn < 0) return mfail("unknown Gmsh element type %lld", (long long)type);
          for (int64_t k = 0; k < n; ++k) {
            int64_t id;
            if (!tk.integer(id)) return mfail("bad element record");
            std::vector<int64_t> nodes(nn);
            for (int q = 0; q < nn; ++q) {
              int64_t nid;
              if (!tk.integer(nid) || !node_index(nid, &nodes[q])) return mfail("element %lld: unknown node", (long long)id);
            }
            if (bte_status st = add_elem(r, (int)type, nodes)) return st;
          }
        }
      }
      tk.next(t);  // $EndElements
      have_elems = true;
    } else if (!t.empty() && t[0] == '$' && t.rfind("$End", 0) != 0) {
      // other sections ($PhysicalNames, $Entities, ...): skip to their end marker
      const std::string end = "$End" + t.substr(1);
      while (tk.next(t) && t != end) {
      }
    }
  }
  if (!have_nodes || !have_elems) return mfail("Gmsh file without $Nodes / $Elements");
  return BTE_OK;
}

// ---- MEDIT: keywords MeshVersionFormatted, Dimension, Vertices n (coords + ref),
//      Triangles / Quadrilaterals / Tetrahedra n (1-based vertices + ref), End
bte_status read_medit(std::istream &in, Raw &r) {
  Tok tk(in, true);
  std::string t;
  int64_t dim = 0;
  bool have_v = false;
  while (tk.next(t)) {
    std::string k = t;
    for (auto &ch : k) ch = (char)std::tolower((unsigned char)ch);
    if (k == "meshversionformatted") {
      int64_t ver;
      if (!tk.integer(ver)) return mfail("bad MeshVersionFormatted");
    } else if (k == "dimension") {
      if (!tk.integer(dim) || (dim != 2 && dim != 3)) return mfail("bad Dimension");
    } else if (k == "vertices") {
      if (dim == 0) return mfail("Vertices before Dimension");
      int64_t n;
      if (!tk.integer(n) || n < 0) return mfail("bad Vertices count");
      r.verts.assign(3 * n, 0.0);
      for (int64_t q = 0; q < n; ++q) {
        for (int a = 0; a < dim; ++a)
          if (!tk.num(r.verts[3 * q + a])) return mfail("bad vertex %lld", (long long)q);
        int64_t ref;
        if (!tk.integer(ref)) return mfail("bad vertex reference");
      }
      have_v = true;
    } else if (k == "triangles" || k == "quadrilaterals" || k == "tetrahedra" || k == "edges" ||
               k == "hexahedra" || k == "prisms" || k == "corners" || k == "ridges" || k == "requiredvertices") {
      int64_t n;
      if (!tk.integer(n) || n < 0) return mfail("bad %s count", t.c_str());
      const int nn = k == "triangles" ? 3 : k == "quadrilaterals" || k == "tetrahedra" ? 4 : k == "edges" ? 2
                   : k == "hexahedra" ? 8 : k == "prisms" ? 6 : 1;
      const bool refs = nn > 1;  // element records end with a reference; corner-type lists do not
      if (k == "prisms" && n > 0)
        return mfail("%s are not supported: tetrahedra, hexahedra, triangles and quadrilaterals only", t.c_str());
      std::vector<int64_t> *dst = k == "triangles" ? &r.tri : k == "quadrilaterals" ? &r.quad
                                : k == "tetrahedra" ? &r.tet : k == "hexahedra" ? &r.hex : nullptr;
      for (int64_t q = 0; q < n; ++q) {
        for (int a = 0; a < nn; ++a) {
          int64_t vid;
          if (!tk.integer(vid)) return mfail("bad %s record", t.c_str());
          if (dst) {
            if (vid < 1) return mfail("%s: vertex index %lld < 1", t.c_str(), (long long)vid);
            dst->push_back(vid - 1);
          }
        }
        if (refs) {
          int64_t ref;
          if (!tk.integer(ref)) return mfail("bad %s reference", t.c_str());
        }
      }
    } else if (k == "end") {
      break;
    } else {
      return mfail("unknown MEDIT keyword '%s'", t.c_str());
    }
  }
  if (!have_v) return mfail("MEDIT file without Vertices");
  r.dim = (int)dim;
  return BTE_OK;
}

}  // namespace

extern "C" {

bte_status bte_mesh_read(const char *path, bte_mesh_data **out) {
  if (!path || !out) return BTE_EINVAL;
  *out = nullptr;
  g_mesh_err.clear();
  std::ifstream f(path);
  if (!f) return mfail("cannot open '%s'", path);
  std::string first;
  f >> first;
  f.seekg(0);
  Raw r;
  bte_status st;
  if (first == "$MeshFormat")
    st = read_gmsh(f, r);
  else
    st = read_medit(f, r);
  if (st) return st;
  const int64_t nv = (int64_t)(r.verts.size() / 3);
  // the cell kind: 3-D when tetrahedra are present (triangles are then boundary
  // tags), else 2-D triangles or quadrilaterals (not both)
  int dim, nvc;
  const std::vector<int64_t> *cells;
  if (!r.tet.empty() && !r.hex.empty()) {
    return mfail("mixed tetrahedra and hexahedra: one cell kind per mesh");
  } else if (!r.tet.empty()) {
    dim = 3, nvc = 4, cells = &r.tet;
  } else if (!r.hex.empty()) {
    dim = 3, nvc = 8, cells = &r.hex;
  } else if (!r.tri.empty() && !r.quad.empty()) {
    return mfail("mixed triangles and quadrilaterals: one cell kind per mesh");
  } else if (!r.tri.empty()) {
    dim = 2, nvc = 3, cells = &r.tri;
  } else if (!r.quad.empty()) {
    dim = 2, nvc = 4, cells = &r.quad;
  } else {
    return mfail("no triangles, quadrilaterals or tetrahedra in '%s'", path);
  }
  if (r.dim == 2 && dim == 3) return mfail("tetrahedra in a 2-D MEDIT mesh");
  for (int64_t v : *cells)
    if (v < 0 || v >= nv) return mfail("vertex index %lld out of range", (long long)v);
  bte_mesh_data *m = new bte_mesh_data;
  m->dim = dim;
  m->nvc = nvc;
  m->nverts = nv;
  m->ncells = (int64_t)(cells->size() / nvc);
  m->verts = new double[r.verts.size()];
  std::copy(r.verts.begin(), r.verts.end(), m->verts);
  m->cells = new int64_t[cells->size()];
  std::copy(cells->begin(), cells->end(), m->cells);
  *out = m;
  return BTE_OK;
}

void bte_mesh_free(bte_mesh_data *m) {
  if (!m) return;
  delete[] m->verts;
  delete[] m->cells;
  delete m;
}

const char *bte_mesh_error(void) { return g_mesh_err.c_str(); }

bte_status bte_partition_rcb(const bte_umesh *mesh, int nparts, int64_t *perm) {
  g_mesh_err.clear();
  if (!mesh || !perm || !mesh->verts || !mesh->cells) return mfail("null argument");
  const int64_t nc = mesh->ncells;
  const int nvc = mesh->nvc > 0 ? mesh->nvc : mesh->dim + 1;
  if (nparts < 1 || nparts > nc) return mfail("nparts %d outside [1, ncells]", nparts);
  if (mesh->dim != 2 && mesh->dim != 3) return mfail("dim must be 2 or 3");
  // centroids: vertex mean in local order
  std::vector<double> cen(3 * (size_t)nc, 0.0);
  for (int64_t c = 0; c < nc; ++c) {
    for (int k = 0; k < nvc; ++k) {
      const int64_t v = mesh->cells[c * nvc + k];
      if (v < 0 || v >= mesh->nverts) return mfail("cell %lld: vertex index out of range", (long long)c);
      for (int a = 0; a < 3; ++a) cen[3 * c + a] += mesh->verts[3 * v + a];
    }
    for (int a = 0; a < 3; ++a) cen[3 * c + a] /= nvc;
  }
  std::vector<int64_t> ids(nc);
  for (int64_t c = 0; c < nc; ++c) ids[c] = c;
  // parts [p0, p1) own cells [lo, hi) of ids; part r ends up with the range
  // [r nc/P, (r+1) nc/P) -- the ranges bte_create_umesh assigns
  auto start = [&](int r) { return (int64_t)((__int128)r * nc / nparts); };
  struct Job { int p0, p1; };
  std::vector<Job> stack{{0, nparts}};
  while (!stack.empty()) {
    const Job j = stack.back();
    stack.pop_back();
    if (j.p1 - j.p0 < 2) continue;
    const int64_t lo = start(j.p0), hi = start(j.p1);
    const int pm = (j.p0 + j.p1) / 2;
    const int64_t mid = start(pm);
    // longest extent of the centroids in this range
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t q = lo; q < hi; ++q)
      for (int a = 0; a < mesh->dim; ++a) {
        mn[a] = std::min(mn[a], cen[3 * ids[q] + a]);
        mx[a] = std::max(mx[a], cen[3 * ids[q] + a]);
      }
    int ax = 0;
    for (int a = 1; a < mesh->dim; ++a)
      if (mx[a] - mn[a] > mx[ax] - mn[ax]) ax = a;
    // split at the (mid - lo)-th smallest coordinate; ties by cell index (deterministic)
    std::nth_element(ids.begin() + lo, ids.begin() + mid, ids.begin() + hi, [&](int64_t a, int64_t b) {
      const double xa = cen[3 * a + ax], xb = cen[3 * b + ax];
      return xa < xb || (xa == xb && a < b);
    });
    stack.push_back({j.p0, pm});
    stack.push_back({pm, j.p1});
  }
  // inside each part keep the input order (canonical order of its cells)
  for (int r = 0; r < nparts; ++r) std::sort(ids.begin() + start(r), ids.begin() + start(r + 1));
  std::copy(ids.begin(), ids.end(), perm);
  return BTE_OK;
}

}  // extern "C"
