// snapshot.cpp -- PMHD1 snapshot write / restart read (the
// "next" row §8f-2 of SURVEY.md).  Format: ASCII header
//   PMHD1 / dims <nx1> <nx2> <nx3> / gamma <g> / time <t> / END
// then little-endian IEEE-754 fp64: the 8 conserved variables over the global
// active grid in variable-major k-j-i order, followed by the global staggered
// b1f (nx1+1 x nx2 x nx3), b2f (nx1 x nx2+1 x nx3), b3f (nx1 x nx2 x nx3+1;
// nx3+1 = 2 layers in 2D) arrays.  The shared face between two blocks is taken
// from the lower block.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "pmhd_host.h"

namespace {

struct G {
  int nx[3], mb[3], nb[3], ng, g3, n[3];
  explicit G(const pmhd_mesh_desc& m) {
    ng = m.ng;
    g3 = (m.nx[2] > 1) ? m.ng : 0;
    for (int a = 0; a < 3; ++a) { nx[a] = m.nx[a]; mb[a] = m.mb[a]; nb[a] = m.nx[a] / m.mb[a]; }
    n[0] = mb[0] + 2 * ng; n[1] = mb[1] + 2 * ng; n[2] = mb[2] + 2 * g3;
  }
  size_t nc() const { return size_t(n[0]) * n[1] * n[2]; }
};

// Visit the global array with extra face layer (ex, ey, ez): fn(gid, local
// index) in global k-j-i order.  A face shared by two blocks is visited once,
// as the upper block's lower face (bitwise equal to the lower block's upper
// face after exchange_ghosts); the domain's last face maps to the last block.
template <class Fn>
void visit(const G& g, int ex, int ey, int ez, Fn&& fn) {
  for (int k = 0; k < g.nx[2] + ez; ++k)
    for (int j = 0; j < g.nx[1] + ey; ++j)
      for (int i = 0; i < g.nx[0] + ex; ++i) {
        const int ci = std::min(i / g.mb[0], g.nb[0] - 1), cj = std::min(j / g.mb[1], g.nb[1] - 1);
        const int ck = std::min(k / g.mb[2], g.nb[2] - 1);
        const int gid = (ck * g.nb[1] + cj) * g.nb[0] + ci;
        const int li = i - ci * g.mb[0] + g.ng, lj = j - cj * g.mb[1] + g.ng;
        const int lk = k - ck * g.mb[2] + g.g3;
        fn(gid, lk, lj, li);
      }
}

}  // namespace

extern "C" {

int pmhd_host_snapshot_write(const char* path, const pmhd_run_config* cfg, double t,
                             double* const* u, double* const* b1f, double* const* b2f,
                             double* const* b3f) {
  const pmhd_mesh_desc& m = cfg->mesh;
  const G g(m);
  std::ofstream f(path, std::ios::binary);
  if (!f) return PMHD_ERR_INPUT;
  char hdr[256];
  std::snprintf(hdr, sizeof(hdr), "PMHD1\ndims %d %d %d\ngamma %.17g\ntime %.17g\nEND\n", m.nx[0],
                m.nx[1], m.nx[2], m.gamma, t);
  f << hdr;
  auto put = [&](double v) { f.write(reinterpret_cast<const char*>(&v), sizeof(v)); };
  const size_t nc = g.nc();
  for (int v = 0; v < 8; ++v)
    visit(g, 0, 0, 0, [&](int b, int k, int j, int i) {
      put(u[b][v * nc + (size_t(k) * g.n[1] + j) * g.n[0] + i]);
    });
  visit(g, 1, 0, 0, [&](int b, int k, int j, int i) {
    put(b1f[b][(size_t(k) * g.n[1] + j) * (g.n[0] + 1) + i]);
  });
  visit(g, 0, 1, 0, [&](int b, int k, int j, int i) {
    put(b2f[b][(size_t(k) * (g.n[1] + 1) + j) * g.n[0] + i]);
  });
  visit(g, 0, 0, 1, [&](int b, int k, int j, int i) {
    put(b3f[b][(size_t(k) * g.n[1] + j) * g.n[0] + i]);
  });
  return f.good() ? PMHD_OK : PMHD_ERR_INPUT;
}

int pmhd_host_snapshot_read(const char* path, const pmhd_run_config* cfg, double* t, double* const* u,
                            double* const* b1f, double* const* b2f, double* const* b3f) {
  const pmhd_mesh_desc& m = cfg->mesh;
  const G g(m);
  std::ifstream f(path, std::ios::binary);
  if (!f) return PMHD_ERR_INPUT;
  std::string line;
  int dims[3] = {0, 0, 0};
  double gamma = 0.0, time = 0.0;
  if (!std::getline(f, line) || line != "PMHD1") return PMHD_ERR_INPUT;
  for (;;) {
    if (!std::getline(f, line)) return PMHD_ERR_INPUT;
    if (line == "END") break;
    std::istringstream ss(line);
    std::string key;
    ss >> key;
    if (key == "dims") ss >> dims[0] >> dims[1] >> dims[2];
    else if (key == "gamma") ss >> gamma;
    else if (key == "time") ss >> time;
    else return PMHD_ERR_INPUT;
  }
  if (dims[0] != m.nx[0] || dims[1] != m.nx[1] || dims[2] != m.nx[2] || gamma != m.gamma)
    return PMHD_ERR_INPUT;
  bool ok = true;
  auto get = [&]() {
    double v = 0.0;
    if (!f.read(reinterpret_cast<char*>(&v), sizeof(v))) ok = false;
    return v;
  };
  const size_t nc = g.nc();
  for (int v = 0; v < 8; ++v)
    visit(g, 0, 0, 0, [&](int b, int k, int j, int i) {
      u[b][v * nc + (size_t(k) * g.n[1] + j) * g.n[0] + i] = get();
    });
  // faces: every block also gets its own upper face (shared with the next
  // block's lower face), so fill both copies of a shared face
  auto put_face = [&](double* const* arr, int dir, int ex, int ey, int ez) {
    visit(g, ex, ey, ez, [&](int b, int k, int j, int i) {
      const double val = get();
      const int n1 = g.n[0] + (dir == 0), n2 = g.n[1] + (dir == 1);
      arr[b][(size_t(k) * n2 + j) * n1 + i] = val;
      const int c[3] = {b % g.nb[0], (b / g.nb[0]) % g.nb[1], b / (g.nb[0] * g.nb[1])};
      const int loc[3] = {i, j, k};
      const int lo = (dir == 2) ? g.g3 : g.ng;
      if (loc[dir] == lo && c[dir] > 0) {  // lower face of block b is the upper face of b-1
        int cc[3] = {c[0], c[1], c[2]};
        cc[dir] -= 1;
        const int bb = (cc[2] * g.nb[1] + cc[1]) * g.nb[0] + cc[0];
        int l2[3] = {i, j, k};
        l2[dir] = lo + g.mb[dir];
        arr[bb][(size_t(l2[2]) * n2 + l2[1]) * n1 + l2[0]] = val;
      }
    });
  };
  put_face(b1f, 0, 1, 0, 0);
  put_face(b2f, 1, 0, 1, 0);
  put_face(b3f, 2, 0, 0, 1);
  if (!ok) return PMHD_ERR_INPUT;
  if (t) *t = time;
  return PMHD_OK;
}

}  // extern "C"
