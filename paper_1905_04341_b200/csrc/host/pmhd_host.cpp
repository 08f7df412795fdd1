// pmhd_host.cpp -- host-side C++ layer above the GPU C-ABI: input files,
// MeshConfig/MeshBlock geometry and problem generators.
//
// Reference interfaces restated here:
//   parse_config
//   MeshConfig / build_mesh   SPEC.md:30-57 (invariants :32-34, errors :53)
//   init_linear_wave       SPEC.md:218-226 (numerical eigenvector, B from a
//                          vector potential so that div B <= 1e-13)
//   WaveSetup              SPEC.md:126-129, background default
// Orszag-Tang, blast and turbulence follow the definitions pinned in
// SURVEY.md §8d (configs M2, M3, M5 of BASELINE.json).
#include "pmhd_host.h"

#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

namespace {

constexpr double kPi = 3.14159265358979323846;

void set_err(char* err, int errlen, const std::string& msg) {
  if (err && errlen > 0) std::snprintf(err, size_t(errlen), "%s", msg.c_str());
}

//---------------------------------------------------------------- geometry
struct Geom {
  int nx[3], mb[3], nb[3], ng, dim, n[3];
  int is, ie, js, je, ks, ke;
  double dx[3], xmin[3];
  explicit Geom(const pmhd_mesh_desc& d) {
    dim = (d.nx[2] == 1) ? 2 : 3;
    ng = d.ng;
    for (int a = 0; a < 3; ++a) {
      nx[a] = d.nx[a]; mb[a] = d.mb[a]; nb[a] = d.nx[a] / d.mb[a];
      xmin[a] = d.xmin[a];
      dx[a] = (d.xmax[a] - d.xmin[a]) / d.nx[a];
      n[a] = mb[a] + 2 * ((a == 2 && dim == 2) ? 0 : ng);
    }
    is = ng; ie = ng + mb[0]; js = ng; je = ng + mb[1];
    if (dim == 3) { ks = ng; ke = ng + mb[2]; } else { ks = 0; ke = 1; }
  }
  void coords(int gid, int c[3]) const {
    c[0] = gid % nb[0]; c[1] = (gid / nb[0]) % nb[1]; c[2] = gid / (nb[0] * nb[1]);
  }
  size_t cidx(int k, int j, int i) const { return (size_t(k) * n[1] + j) * n[0] + i; }
  size_t f1(int k, int j, int i) const { return (size_t(k) * n[1] + j) * (n[0] + 1) + i; }
  size_t f2(int k, int j, int i) const { return (size_t(k) * (n[1] + 1) + j) * n[0] + i; }
  size_t f3(int k, int j, int i) const { return (size_t(k) * n[1] + j) * n[0] + i; }
  size_t ncell() const { return size_t(n[0]) * n[1] * n[2]; }
  // global coordinate of a local cell face (lo=true) or centre
  double xf(int a, int c0, int loc) const {  // face at local index loc (lower face of cell loc)
    const int s = (a == 0) ? is : (a == 1 ? js : ks);
    return xmin[a] + double(c0 * mb[a] + (loc - s)) * dx[a];
  }
  double xc(int a, int c0, int loc) const {
    const int s = (a == 0) ? is : (a == 1 ? js : ks);
    return xmin[a] + (double(c0 * mb[a] + (loc - s)) + 0.5) * dx[a];
  }
};

//---------------------------------------------------------------- eigen
// 1-D ideal-MHD flux of the conserved wave-frame state
// U = (d, mn, mt1, mt2, E, bt1, bt2) with fixed normal field bn.
template <class T>
void flux1d(const T* U, double bn, double gamma, T* F) {
  const T d = U[0], vn = U[1] / d, vt1 = U[2] / d, vt2 = U[3] / d;
  const T bt1 = U[5], bt2 = U[6];
  const T pb = 0.5 * (bn * bn + bt1 * bt1 + bt2 * bt2);
  const T p = (gamma - 1.0) * (U[4] - 0.5 * (U[1] * vn + U[2] * vt1 + U[3] * vt2) - pb);
  const T pt = p + pb;
  F[0] = U[1];
  F[1] = U[1] * vn + pt - bn * bn;
  F[2] = U[2] * vn - bn * bt1;
  F[3] = U[3] * vn - bn * bt2;
  F[4] = (U[4] + pt) * vn - bn * (vn * bn + vt1 * bt1 + vt2 * bt2);
  F[5] = bt1 * vn - bn * vt1;
  F[6] = bt2 * vn - bn * vt2;
}

// Complex-step Jacobian dF/dU (exact to round-off; no subtractive error).
void jacobian(const double* U, double bn, double gamma, double J[7][7]) {
  const double h = 1e-30;
  for (int c = 0; c < 7; ++c) {
    std::complex<double> Uc[7], Fc[7];
    for (int r = 0; r < 7; ++r) Uc[r] = U[r];
    Uc[c] += std::complex<double>(0.0, h);
    flux1d(Uc, bn, gamma, Fc);
    for (int r = 0; r < 7; ++r) J[r][c] = Fc[r].imag() / h;
  }
}

// Solve A x = b (7x7) by Gaussian elimination with partial pivoting.
bool solve7(double A[7][7], double* b) {
  for (int c = 0; c < 7; ++c) {
    int p = c;
    for (int r = c + 1; r < 7; ++r) if (std::fabs(A[r][c]) > std::fabs(A[p][c])) p = r;
    if (A[p][c] == 0.0) A[p][c] = 1e-300;
    if (p != c) { for (int k = 0; k < 7; ++k) std::swap(A[c][k], A[p][k]); std::swap(b[c], b[p]); }
    for (int r = c + 1; r < 7; ++r) {
      const double f = A[r][c] / A[c][c];
      for (int k = c; k < 7; ++k) A[r][k] -= f * A[c][k];
      b[r] -= f * b[c];
    }
  }
  for (int c = 6; c >= 0; --c) {
    double s = b[c];
    for (int k = c + 1; k < 7; ++k) s -= A[c][k] * b[k];
    b[c] = s / A[c][c];
  }
  return true;
}

struct WaveEigen {
  double lambda, r[7], residual;
  double n[3], t1[3], t2[3];  // wave frame (lab components)
  double k[3], kmag;          // wavevector (rad / length)
  double U0[7];               // background, wave frame conserved
  double bn;
};

void cross(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

int wave_eigen(const pmhd_run_config& cfg, WaveEigen& W) {
  const pmhd_mesh_desc& d = cfg.mesh;
  double L[3];
  for (int a = 0; a < 3; ++a) L[a] = d.xmax[a] - d.xmin[a];
  for (int a = 0; a < 3; ++a) W.k[a] = 2.0 * kPi * cfg.wave_n[a] / L[a];
  W.kmag = std::sqrt(W.k[0] * W.k[0] + W.k[1] * W.k[1] + W.k[2] * W.k[2]);
  if (!(W.kmag > 0.0)) return PMHD_ERR_CONFIG;
  for (int a = 0; a < 3; ++a) W.n[a] = W.k[a] / W.kmag;
  const double z[3] = {0.0, 0.0, 1.0};
  double t1[3];
  cross(z, W.n, t1);
  double t1m = std::sqrt(t1[0] * t1[0] + t1[1] * t1[1] + t1[2] * t1[2]);
  if (t1m < 1e-12) { t1[0] = 1.0; t1[1] = 0.0; t1[2] = 0.0; t1m = 1.0; }
  for (int a = 0; a < 3; ++a) W.t1[a] = t1[a] / t1m;
  cross(W.n, W.t1, W.t2);

  const double rho = cfg.wave_rho, p = cfg.wave_p, g = d.gamma;
  const double vn = cfg.wave_v[0], vt1 = cfg.wave_v[1], vt2 = cfg.wave_v[2];
  const double bn = cfg.wave_b[0], bt1 = cfg.wave_b[1], bt2 = cfg.wave_b[2];
  W.bn = bn;
  W.U0[0] = rho; W.U0[1] = rho * vn; W.U0[2] = rho * vt1; W.U0[3] = rho * vt2;
  W.U0[4] = p / (g - 1.0) + 0.5 * rho * (vn * vn + vt1 * vt1 + vt2 * vt2) +
            0.5 * (bn * bn + bt1 * bt1 + bt2 * bt2);
  W.U0[5] = bt1; W.U0[6] = bt2;

  // characteristic speeds (numerical values; the eigenvector comes from the
  // Jacobian, not from hand-coded formulas)
  const double asq = g * p / rho, bsq = (bn * bn + bt1 * bt1 + bt2 * bt2) / rho, cax2 = bn * bn / rho;
  const double disc = std::sqrt(std::fmax(0.0, (asq + bsq) * (asq + bsq) - 4.0 * asq * cax2));
  const double cf = std::sqrt(0.5 * (asq + bsq + disc));
  const double cs = std::sqrt(std::fmax(0.0, 0.5 * (asq + bsq - disc)));
  const double ca = std::sqrt(cax2);
  const double speeds[7] = {vn - cf, vn - ca, vn - cs, vn, vn + cs, vn + ca, vn + cf};
  if (cfg.wave_mode < 0 || cfg.wave_mode > 6) return PMHD_ERR_CONFIG;
  const double lam = speeds[cfg.wave_mode];

  double J[7][7];
  jacobian(W.U0, bn, g, J);
  // inverse iteration with the (numerical) eigenvalue as shift
  double x[7];
  for (int r = 0; r < 7; ++r) x[r] = 1.0 + 0.1 * r;
  const double shift = lam + 1e-9 * (1.0 + std::fabs(lam));
  for (int it = 0; it < 6; ++it) {
    double A[7][7];
    for (int r = 0; r < 7; ++r)
      for (int c = 0; c < 7; ++c) A[r][c] = J[r][c] - (r == c ? shift : 0.0);
    solve7(A, x);
    double nrm = 0.0;
    for (int r = 0; r < 7; ++r) nrm += x[r] * x[r];
    nrm = std::sqrt(nrm);
    for (int r = 0; r < 7; ++r) x[r] /= nrm;
  }
  // deterministic sign: largest component positive
  int im = 0;
  for (int r = 1; r < 7; ++r) if (std::fabs(x[r]) > std::fabs(x[im]) + 1e-12) im = r;
  if (x[im] < 0.0) for (int r = 0; r < 7; ++r) x[r] = -x[r];
  // Rayleigh-type refinement of lambda and residual
  double Jx[7];
  for (int r = 0; r < 7; ++r) { Jx[r] = 0.0; for (int c = 0; c < 7; ++c) Jx[r] += J[r][c] * x[c]; }
  double num = 0.0, den = 0.0;
  for (int r = 0; r < 7; ++r) { num += Jx[r] * x[r]; den += x[r] * x[r]; }
  W.lambda = num / den;
  double res = 0.0;
  for (int r = 0; r < 7; ++r) res = std::fmax(res, std::fabs(Jx[r] - W.lambda * x[r]));
  W.residual = res;
  for (int r = 0; r < 7; ++r) W.r[r] = x[r];
  return PMHD_OK;
}

// Background + perturbation in LAB components at phase theta.
void wave_state(const pmhd_run_config& cfg, const WaveEigen& W, double theta, double* q8) {
  const double A = cfg.wave_amp, cs = std::cos(theta);
  const double dU[7] = {W.U0[0] + A * W.r[0] * cs, W.U0[1] + A * W.r[1] * cs,
                        W.U0[2] + A * W.r[2] * cs, W.U0[3] + A * W.r[3] * cs,
                        W.U0[4] + A * W.r[4] * cs, W.U0[5] + A * W.r[5] * cs,
                        W.U0[6] + A * W.r[6] * cs};
  q8[0] = dU[0];
  for (int a = 0; a < 3; ++a) {
    q8[1 + a] = dU[1] * W.n[a] + dU[2] * W.t1[a] + dU[3] * W.t2[a];
    q8[5 + a] = W.bn * W.n[a] + dU[5] * W.t1[a] + dU[6] * W.t2[a];
  }
  q8[4] = dU[4];
}

// Vector potential of the B perturbation: A_vec = amp (b x k)/|k|^2 sin(k.x),
// b = r5 t1 + r6 t2 (perpendicular to k), so curl A = amp b cos(k.x).
void wave_vecpot(const pmhd_run_config& cfg, const WaveEigen& W, const double* x, double* Av) {
  double b[3], bxk[3];
  for (int a = 0; a < 3; ++a) b[a] = W.r[5] * W.t1[a] + W.r[6] * W.t2[a];
  cross(b, W.k, bxk);
  const double ph = W.k[0] * x[0] + W.k[1] * x[1] + W.k[2] * x[2];
  const double s = cfg.wave_amp * std::sin(ph) / (W.kmag * W.kmag);
  for (int a = 0; a < 3; ++a) Av[a] = bxk[a] * s;
}

//---------------------------------------------------------------- face fill helpers
// Fills faces from a vector potential Avec(x) given at edges, plus a uniform
// background B0.  Discretely divergence free to round-off.
template <class AFn>
void faces_from_vecpot(const Geom& G, const int c[3], const double* B0, AFn&& Afn, double* b1f,
                       double* b2f, double* b3f) {
  const bool d3 = G.dim == 3;
  const int kend = d3 ? G.ke : G.ke;  // cells
  auto A = [&](double x, double y, double z, int comp) {
    double p[3] = {x, y, z}, a[3];
    Afn(p, a);
    return a[comp];
  };
  for (int k = G.ks; k < kend; ++k)
    for (int j = G.js; j < G.je; ++j)
      for (int i = G.is; i <= G.ie; ++i) {  // b1f at (x_{i-1/2}, y_j, z_k)
        const double x = G.xf(0, c[0], i), yc = G.xc(1, c[1], j), zc = d3 ? G.xc(2, c[2], k) : 0.0;
        const double ym = G.xf(1, c[1], j), yp = G.xf(1, c[1], j + 1);
        double v = B0[0] + (A(x, yp, zc, 2) - A(x, ym, zc, 2)) / G.dx[1];
        if (d3) {
          const double zm = G.xf(2, c[2], k), zp = G.xf(2, c[2], k + 1);
          v -= (A(x, yc, zp, 1) - A(x, yc, zm, 1)) / G.dx[2];
        }
        b1f[G.f1(k, j, i)] = v;
      }
  for (int k = G.ks; k < kend; ++k)
    for (int j = G.js; j <= G.je; ++j)
      for (int i = G.is; i < G.ie; ++i) {  // b2f at (x_i, y_{j-1/2}, z_k)
        const double xc = G.xc(0, c[0], i), y = G.xf(1, c[1], j), zc = d3 ? G.xc(2, c[2], k) : 0.0;
        const double xm = G.xf(0, c[0], i), xp = G.xf(0, c[0], i + 1);
        double v = B0[1] - (A(xp, y, zc, 2) - A(xm, y, zc, 2)) / G.dx[0];
        if (d3) {
          const double zm = G.xf(2, c[2], k), zp = G.xf(2, c[2], k + 1);
          v += (A(xc, y, zp, 0) - A(xc, y, zm, 0)) / G.dx[2];
        }
        b2f[G.f2(k, j, i)] = v;
      }
  const int k3end = d3 ? G.ke + 1 : 2;
  for (int k = G.ks; k < k3end; ++k)
    for (int j = G.js; j < G.je; ++j)
      for (int i = G.is; i < G.ie; ++i) {  // b3f at (x_i, y_j, z_{k-1/2})
        const double xc = G.xc(0, c[0], i), yc = G.xc(1, c[1], j);
        const double z = d3 ? G.xf(2, c[2], k) : 0.0;
        const double xm = G.xf(0, c[0], i), xp = G.xf(0, c[0], i + 1);
        const double ym = G.xf(1, c[1], j), yp = G.xf(1, c[1], j + 1);
        const double v = B0[2] + (A(xp, yc, z, 1) - A(xm, yc, z, 1)) / G.dx[0] -
                         (A(xc, yp, z, 0) - A(xc, ym, z, 0)) / G.dx[1];
        b3f[G.f3(k, j, i)] = v;
      }
}

void uniform_faces(const Geom& G, const double* B0, double* b1f, double* b2f, double* b3f) {
  const int k3end = (G.dim == 3) ? G.ke + 1 : 2;
  for (int k = G.ks; k < G.ke; ++k)
    for (int j = G.js; j < G.je; ++j)
      for (int i = G.is; i <= G.ie; ++i) b1f[G.f1(k, j, i)] = B0[0];
  for (int k = G.ks; k < G.ke; ++k)
    for (int j = G.js; j <= G.je; ++j)
      for (int i = G.is; i < G.ie; ++i) b2f[G.f2(k, j, i)] = B0[1];
  for (int k = G.ks; k < k3end; ++k)
    for (int j = G.js; j < G.je; ++j)
      for (int i = G.is; i < G.ie; ++i) b3f[G.f3(k, j, i)] = B0[2];
}

// Cell-centred field from the faces + total energy from (rho, v, p).
void finish_cells(const Geom& G, double gamma, double* u, const double* b1f, const double* b2f,
                  const double* b3f, const std::vector<double>& pgas) {
  const size_t nc = G.ncell();
  size_t n = 0;
  for (int k = G.ks; k < G.ke; ++k)
    for (int j = G.js; j < G.je; ++j)
      for (int i = G.is; i < G.ie; ++i, ++n) {
        const size_t c = G.cidx(k, j, i);
        const double B1 = 0.5 * (b1f[G.f1(k, j, i)] + b1f[G.f1(k, j, i + 1)]);
        const double B2 = 0.5 * (b2f[G.f2(k, j, i)] + b2f[G.f2(k, j + 1, i)]);
        const double B3 = 0.5 * (b3f[G.f3(k, j, i)] + b3f[G.f3(k + 1, j, i)]);
        u[5 * nc + c] = B1; u[6 * nc + c] = B2; u[7 * nc + c] = B3;
        if (!pgas.empty()) {
          const double d = u[c];
          const double ke = 0.5 * (u[nc + c] * u[nc + c] + u[2 * nc + c] * u[2 * nc + c] +
                                   u[3 * nc + c] * u[3 * nc + c]) / d;
          u[4 * nc + c] = pgas[n] / (gamma - 1.0) + ke + 0.5 * (B1 * B1 + B2 * B2 + B3 * B3);
        }
      }
}

uint64_t g_dummy = 0;

double u01(std::mt19937_64& rng) { return double(rng() >> 11) * (1.0 / 9007199254740992.0); }

struct TurbMode { int k[3]; double a[3]; double phase; };

// Solenoidal Fourier velocity modes, |k| in [1,2] (integer k, half space so
// the modes are orthogonal), amplitudes/phases from mt19937_64(seed) drawn in
// a fixed (kx,ky,kz) loop order; normalised analytically to rms Mach.
std::vector<TurbMode> turb_modes(const pmhd_run_config& cfg, double* scale) {
  std::mt19937_64 rng(cfg.turb_seed);
  std::vector<TurbMode> modes;
  const bool d3 = cfg.mesh.nx[2] > 1;
  double s2 = 0.0;
  for (int kx = -2; kx <= 2; ++kx)
    for (int ky = -2; ky <= 2; ++ky)
      for (int kz = -2; kz <= 2; ++kz) {
        if (!d3 && kz != 0) continue;
        const int k2 = kx * kx + ky * ky + kz * kz;
        if (k2 < 1 || k2 > 4) continue;
        const bool half = (kx > 0) || (kx == 0 && ky > 0) || (kx == 0 && ky == 0 && kz > 0);
        if (!half) continue;
        TurbMode m;
        m.k[0] = kx; m.k[1] = ky; m.k[2] = kz;
        double a[3] = {2.0 * u01(rng) - 1.0, 2.0 * u01(rng) - 1.0, 2.0 * u01(rng) - 1.0};
        m.phase = 2.0 * kPi * u01(rng);
        const double ak = (a[0] * kx + a[1] * ky + a[2] * kz) / double(k2);
        for (int c = 0; c < 3; ++c) m.a[c] = a[c] - ak * m.k[c];
        s2 += 0.5 * (m.a[0] * m.a[0] + m.a[1] * m.a[1] + m.a[2] * m.a[2]);
        modes.push_back(m);
      }
  const double cs = std::sqrt(cfg.mesh.gamma * cfg.uniform_w[4] / cfg.uniform_w[0]);
  *scale = cfg.turb_mach * cs / std::sqrt(s2);
  return modes;
}

//---------------------------------------------------------------- config parse
std::string trim(const std::string& s) {
  size_t a = s.find_first_not_of(" \t\r"), b = s.find_last_not_of(" \t\r");
  if (a == std::string::npos) return "";
  return s.substr(a, b - a + 1);
}

bool parse_int(const std::string& v, int* out) {
  char* end = nullptr;
  long x = std::strtol(v.c_str(), &end, 10);
  if (end == v.c_str() || *end != '\0') return false;
  *out = int(x);
  return true;
}
bool parse_dbl(const std::string& v, double* out) {
  char* end = nullptr;
  double x = std::strtod(v.c_str(), &end);
  if (end == v.c_str() || *end != '\0') return false;
  *out = x;
  return true;
}

}  // namespace

extern "C" {

void pmhd_host_config_defaults(pmhd_run_config* c) {
  std::memset(c, 0, sizeof(*c));
  pmhd_mesh_desc& m = c->mesh;
  for (int a = 0; a < 3; ++a) { m.nx[a] = 16; m.mb[a] = 16; m.xmin[a] = 0.0; m.xmax[a] = 1.0; }
  m.ng = 2;
  m.gamma = 5.0 / 3.0;
  m.cfl = 0.3;
  m.riemann = PMHD_RIEMANN_HLLD;
  m.limiter = PMHD_LIMITER_MC;
  m.eos_mode = PMHD_EOS_ERROR;
  m.emf_mode = PMHD_EMF_UPWIND;
  m.dfloor = std::sqrt(1024.0 * 1.17549435082228750797e-38);  // sqrt(1024 FLT_MIN)
  m.pfloor = m.dfloor;
  c->pgen = PMHD_PGEN_LINEAR_WAVE;
  c->wave_amp = 1e-6;
  c->wave_n[0] = 1; c->wave_n[1] = 0; c->wave_n[2] = 0;
  c->wave_mode = 6;
  c->wave_rho = 1.0; c->wave_p = 0.6;
  c->wave_b[0] = 1.0; c->wave_b[1] = std::sqrt(2.0); c->wave_b[2] = 0.5;
  c->blast_pin = 10.0; c->blast_pout = 0.1; c->blast_r = 0.1; c->blast_rho = 1.0;
  c->blast_b[0] = 1.0 / std::sqrt(2.0); c->blast_b[1] = 1.0 / std::sqrt(2.0); c->blast_b[2] = 0.0;
  c->turb_mach = 1.0;
  c->turb_seed = 1905043410ULL;
  c->turb_drive = 0;
  c->turb_dedt = 1.0;
  c->turb_every = 1;
  c->uniform_w[0] = 1.0; c->uniform_w[4] = 0.6;
  c->uniform_w[5] = std::sqrt(0.6);
  c->nlim = -1;
  c->tlim = 0.0;
  c->workers = 1;
  c->gpus = 1;
}

int pmhd_host_config_parse(const char* text, pmhd_run_config* c, int* err_line, char* err,
                           int errlen) {
  if (err_line) *err_line = 0;
  std::string all = text ? text : "";
  size_t pos = 0;
  int line = 0;
  while (pos <= all.size()) {
    size_t nl = all.find('\n', pos);
    if (nl == std::string::npos) nl = all.size();
    std::string ln = all.substr(pos, nl - pos);
    pos = nl + 1;
    ++line;
    const size_t hash = ln.find('#');
    if (hash != std::string::npos) ln = ln.substr(0, hash);
    ln = trim(ln);
    if (ln.empty()) { if (nl == all.size()) break; continue; }
    if (ln.front() == '<' && ln.back() == '>') continue;  // Athena++ <block> headers
    const size_t eq = ln.find('=');
    auto fail = [&](const std::string& msg) {
      if (err_line) *err_line = line;
      set_err(err, errlen, "line " + std::to_string(line) + ": " + msg);
      return PMHD_ERR_INPUT;
    };
    if (eq == std::string::npos) return fail("expected 'key = value'");
    const std::string key = trim(ln.substr(0, eq)), val = trim(ln.substr(eq + 1));
    pmhd_mesh_desc& m = c->mesh;
    bool ok = true;
    int ival;
    double dval;
    auto I = [&](int* dst) { ok = parse_int(val, &ival); if (ok) *dst = ival; };
    auto D = [&](double* dst) { ok = parse_dbl(val, &dval); if (ok) *dst = dval; };
    if (key == "nx1") I(&m.nx[0]); else if (key == "nx2") I(&m.nx[1]); else if (key == "nx3") I(&m.nx[2]);
    else if (key == "mb1") I(&m.mb[0]); else if (key == "mb2") I(&m.mb[1]); else if (key == "mb3") I(&m.mb[2]);
    else if (key == "ng") I(&m.ng);
    else if (key == "x1min") D(&m.xmin[0]); else if (key == "x1max") D(&m.xmax[0]);
    else if (key == "x2min") D(&m.xmin[1]); else if (key == "x2max") D(&m.xmax[1]);
    else if (key == "x3min") D(&m.xmin[2]); else if (key == "x3max") D(&m.xmax[2]);
    else if (key == "gamma") D(&m.gamma);
    else if (key == "cfl" || key == "cfl_number") D(&m.cfl);
    else if (key == "dfloor") D(&m.dfloor);
    else if (key == "pfloor") D(&m.pfloor);
    else if (key == "riemann") {
      if (val == "hlld") m.riemann = PMHD_RIEMANN_HLLD;
      else if (val == "hlle") m.riemann = PMHD_RIEMANN_HLLE;
      else if (val == "roe") m.riemann = PMHD_RIEMANN_ROE;
      else ok = false;
    } else if (key == "limiter") {
      if (val == "mc") m.limiter = PMHD_LIMITER_MC; else if (val == "vanleer") m.limiter = PMHD_LIMITER_VANLEER; else ok = false;
    } else if (key == "eos_mode") {
      if (val == "error") m.eos_mode = PMHD_EOS_ERROR; else if (val == "floor") m.eos_mode = PMHD_EOS_FLOOR; else ok = false;
    } else if (key == "emf") {
      if (val == "upwind") m.emf_mode = PMHD_EMF_UPWIND; else if (val == "arith") m.emf_mode = PMHD_EMF_ARITH; else ok = false;
    } else if (key == "pgen" || key == "problem") {
      if (val == "linear_wave") c->pgen = PMHD_PGEN_LINEAR_WAVE;
      else if (val == "orszag_tang") c->pgen = PMHD_PGEN_ORSZAG_TANG;
      else if (val == "blast") c->pgen = PMHD_PGEN_BLAST;
      else if (val == "turbulence") c->pgen = PMHD_PGEN_TURBULENCE;
      else if (val == "uniform") c->pgen = PMHD_PGEN_UNIFORM;
      else ok = false;
    } else if (key == "wave_amp" || key == "amp") D(&c->wave_amp);
    else if (key == "wave_n1") I(&c->wave_n[0]); else if (key == "wave_n2") I(&c->wave_n[1]);
    else if (key == "wave_n3") I(&c->wave_n[2]);
    else if (key == "wave_mode" || key == "wave_flag") {
      if (val == "fast") c->wave_mode = 6; else if (val == "alfven") c->wave_mode = 5;
      else if (val == "slow") c->wave_mode = 4; else if (val == "entropy") c->wave_mode = 3;
      else { I(&c->wave_mode); if (ok && (c->wave_mode < 0 || c->wave_mode > 6)) ok = false; }
    } else if (key == "wave_rho") D(&c->wave_rho); else if (key == "wave_p") D(&c->wave_p);
    else if (key == "wave_vn") D(&c->wave_v[0]); else if (key == "wave_vt1") D(&c->wave_v[1]);
    else if (key == "wave_vt2") D(&c->wave_v[2]);
    else if (key == "wave_bn") D(&c->wave_b[0]); else if (key == "wave_bt1") D(&c->wave_b[1]);
    else if (key == "wave_bt2") D(&c->wave_b[2]);
    else if (key == "blast_pin") D(&c->blast_pin); else if (key == "blast_pout") D(&c->blast_pout);
    else if (key == "blast_r") D(&c->blast_r); else if (key == "blast_rho") D(&c->blast_rho);
    else if (key == "blast_b1") D(&c->blast_b[0]); else if (key == "blast_b2") D(&c->blast_b[1]);
    else if (key == "blast_b3") D(&c->blast_b[2]);
    else if (key == "turb_mach") D(&c->turb_mach);
    else if (key == "turb_seed") { double s; D(&s); if (ok) c->turb_seed = (uint64_t)s; }
    else if (key == "turb_drive") I(&c->turb_drive);
    else if (key == "turb_dedt") D(&c->turb_dedt);
    else if (key == "turb_every") I(&c->turb_every);
    else if (key == "rho") D(&c->uniform_w[0]);
    else if (key == "v1") D(&c->uniform_w[1]); else if (key == "v2") D(&c->uniform_w[2]);
    else if (key == "v3") D(&c->uniform_w[3]); else if (key == "p") D(&c->uniform_w[4]);
    else if (key == "b1") D(&c->uniform_w[5]); else if (key == "b2") D(&c->uniform_w[6]);
    else if (key == "b3") D(&c->uniform_w[7]);
    else if (key == "nlim") I(&c->nlim);
    else if (key == "tlim") D(&c->tlim);
    else if (key == "workers") I(&c->workers);
    else if (key == "gpus") I(&c->gpus);
    else if (key == "policy") {  // CPU loop pattern (exec_engine); GPU ignores it
      if (!(val == "simd_nested" || val == "mdrange" || val == "flat1d" || val == "tiled_team")) ok = false;
    } else return fail("unknown key '" + key + "'");
    if (!ok) return fail("malformed value '" + val + "' for key '" + key + "'");
    if (nl == all.size()) break;
  }
  return PMHD_OK;
}

int pmhd_host_validate(const pmhd_run_config* c, char* err, int errlen) {
  const pmhd_mesh_desc& m = c->mesh;
  if (m.ng < 2 || m.ng > 4) { set_err(err, errlen, "ng must be in [2, 4]"); return PMHD_ERR_CONFIG; }
  for (int a = 0; a < 3; ++a) {
    if (m.nx[a] < 1 || m.mb[a] < 1) { set_err(err, errlen, "cell counts must be positive"); return PMHD_ERR_CONFIG; }
    if (m.nx[a] % m.mb[a]) {
      set_err(err, errlen, "nx" + std::to_string(a + 1) + " not divisible by mb" + std::to_string(a + 1));
      return PMHD_ERR_CONFIG;
    }
    if (!(m.xmax[a] > m.xmin[a])) { set_err(err, errlen, "empty domain"); return PMHD_ERR_CONFIG; }
  }
  if (m.nx[1] == 1) { set_err(err, errlen, "1D meshes are not supported"); return PMHD_ERR_CONFIG; }
  // a block must be wider than its ghost layer so that exchange reads and
  // ghost writes never overlap
  if ((m.nx[2] > 1 && m.mb[2] <= m.ng) || m.mb[0] <= m.ng || m.mb[1] <= m.ng) {
    set_err(err, errlen, "meshblock must have more than ng cells per dimension");
    return PMHD_ERR_CONFIG;
  }
  if (!(m.gamma > 1.0)) { set_err(err, errlen, "gamma must be > 1"); return PMHD_ERR_CONFIG; }
  if (!(m.cfl > 0.0 && m.cfl < 1.0)) { set_err(err, errlen, "cfl must be in (0,1)"); return PMHD_ERR_CONFIG; }
  if (c->turb_drive && (c->turb_every < 1 || !(c->turb_dedt >= 0.0))) {
    set_err(err, errlen, "turb_every must be >= 1 and turb_dedt >= 0");
    return PMHD_ERR_CONFIG;
  }
  return PMHD_OK;
}

//---------------------------------------------------------- turbulence driving
int pmhd_host_drive_modes(const pmhd_run_config* cfg, long long event, pmhd_drive_modes* out) {
  if (!cfg || !out || event < 0) return PMHD_ERR_INPUT;
  std::mt19937_64 rng(cfg->turb_seed ^ (0x9E3779B97F4A7C15ULL * (uint64_t)(event + 1)));
  const bool d3 = cfg->mesh.nx[2] > 1;
  out->n = 0;
  for (int kx = -2; kx <= 2; ++kx)
    for (int ky = -2; ky <= 2; ++ky)
      for (int kz = -2; kz <= 2; ++kz) {
        if (!d3 && kz != 0) continue;
        const int k2 = kx * kx + ky * ky + kz * kz;
        if (k2 < 1 || k2 > 4) continue;
        const bool half = (kx > 0) || (kx == 0 && ky > 0) || (kx == 0 && ky == 0 && kz > 0);
        if (!half) continue;
        const int m = out->n++;
        const int k[3] = {kx, ky, kz};
        double c[3], sn[3];
        for (int a = 0; a < 3; ++a) c[a] = 2.0 * u01(rng) - 1.0;
        for (int a = 0; a < 3; ++a) sn[a] = 2.0 * u01(rng) - 1.0;
        const double ck = (c[0] * kx + c[1] * ky + c[2] * kz) / double(k2);
        const double sk = (sn[0] * kx + sn[1] * ky + sn[2] * kz) / double(k2);
        for (int a = 0; a < 3; ++a) {
          out->k[m][a] = k[a];
          out->c[m][a] = c[a] - ck * k[a];
          out->s[m][a] = sn[a] - sk * k[a];
        }
      }
  return PMHD_OK;
}

int pmhd_host_drive_tables(const pmhd_run_config* cfg, int axis, double* cos_tab, double* sin_tab) {
  if (!cfg || axis < 0 || axis > 2 || !cos_tab || !sin_tab) return PMHD_ERR_INPUT;
  const int n = cfg->mesh.nx[axis];
  for (int k = -2; k <= 2; ++k)
    for (int g = 0; g < n; ++g) {
      // phase of wavenumber k at the centre of global cell g (domain-relative,
      // so the tables do not depend on the extent)
      const double th = 2.0 * kPi * double(k) * (double(g) + 0.5) / double(n);
      cos_tab[(k + 2) * n + g] = std::cos(th);
      sin_tab[(k + 2) * n + g] = std::sin(th);
    }
  return PMHD_OK;
}

double pmhd_host_drive_scale(double a, double b, double de) {
  if (!(a > 0.0) || !(de > 0.0)) return 0.0;
  return (-b + std::sqrt(b * b + 4.0 * a * de)) / (2.0 * a);
}

int pmhd_host_nblocks(const pmhd_run_config* c) {
  const pmhd_mesh_desc& m = c->mesh;
  return (m.nx[0] / m.mb[0]) * (m.nx[1] / m.mb[1]) * (m.nx[2] / m.mb[2]);
}

void pmhd_host_block_dims(const pmhd_run_config* c, int n[3]) {
  Geom G(c->mesh);
  n[0] = G.n[0]; n[1] = G.n[1]; n[2] = G.n[2];
}

void pmhd_host_block_coords(const pmhd_run_config* c, int gid, int out[3]) {
  Geom G(c->mesh);
  G.coords(gid, out);
}

int pmhd_host_wave_eigen(const pmhd_run_config* c, double* lambda, double r[7], double* residual) {
  WaveEigen W;
  const int rc = wave_eigen(*c, W);
  if (rc) return rc;
  if (lambda) *lambda = W.lambda;
  if (r) for (int n = 0; n < 7; ++n) r[n] = W.r[n];
  if (residual) *residual = W.residual;
  return PMHD_OK;
}

double pmhd_host_default_tlim(const pmhd_run_config* c) {
  if (c->tlim > 0.0) return c->tlim;
  if (c->pgen == PMHD_PGEN_LINEAR_WAVE) {
    WaveEigen W;
    if (wave_eigen(*c, W)) return 1.0;
    return 2.0 * kPi / (W.kmag * std::fabs(W.lambda));  // one period
  }
  if (c->pgen == PMHD_PGEN_ORSZAG_TANG) return 0.5;
  if (c->pgen == PMHD_PGEN_BLAST) return 0.2;
  return 1.0;
}

int pmhd_host_pgen_block(const pmhd_run_config* cfg, int gid, double* u, double* b1f, double* b2f,
                         double* b3f) {
  char e[128];
  if (pmhd_host_validate(cfg, e, sizeof(e))) return PMHD_ERR_CONFIG;
  const Geom G(cfg->mesh);
  int c[3];
  G.coords(gid, c);
  const size_t nc = G.ncell();
  const double gamma = cfg->mesh.gamma;
  std::vector<double> pgas;
  const bool d3 = G.dim == 3;

  switch (cfg->pgen) {
    case PMHD_PGEN_LINEAR_WAVE: {
      WaveEigen W;
      if (wave_eigen(*cfg, W)) return PMHD_ERR_CONFIG;
      for (int k = G.ks; k < G.ke; ++k)
        for (int j = G.js; j < G.je; ++j)
          for (int i = G.is; i < G.ie; ++i) {
            const double x = G.xc(0, c[0], i), y = G.xc(1, c[1], j), z = d3 ? G.xc(2, c[2], k) : 0.0;
            double q[8];
            wave_state(*cfg, W, W.k[0] * x + W.k[1] * y + W.k[2] * z, q);
            const size_t ci = G.cidx(k, j, i);
            for (int v = 0; v < 5; ++v) u[v * nc + ci] = q[v];
          }
      double B0[3];
      for (int a = 0; a < 3; ++a) B0[a] = W.bn * W.n[a] + W.U0[5] * W.t1[a] + W.U0[6] * W.t2[a];
      faces_from_vecpot(G, c, B0, [&](const double* x, double* A) { wave_vecpot(*cfg, W, x, A); },
                        b1f, b2f, b3f);
      finish_cells(G, gamma, u, b1f, b2f, b3f, pgas);
      break;
    }
    case PMHD_PGEN_ORSZAG_TANG: {  // 2D/3D-extruded vortex
      const double d0 = 25.0 / (36.0 * kPi), p0 = 5.0 / (12.0 * kPi), B0 = 1.0 / std::sqrt(4.0 * kPi);
      for (int k = G.ks; k < G.ke; ++k)
        for (int j = G.js; j < G.je; ++j)
          for (int i = G.is; i < G.ie; ++i) {
            const double x = G.xc(0, c[0], i), y = G.xc(1, c[1], j);
            const size_t ci = G.cidx(k, j, i);
            u[ci] = d0;
            u[nc + ci] = -d0 * std::sin(2.0 * kPi * y);
            u[2 * nc + ci] = d0 * std::sin(2.0 * kPi * x);
            u[3 * nc + ci] = 0.0;
            pgas.push_back(p0);
          }
      const double zero[3] = {0.0, 0.0, 0.0};
      faces_from_vecpot(G, c, zero, [&](const double* x, double* A) {
        A[0] = 0.0; A[1] = 0.0;
        A[2] = B0 * (std::cos(4.0 * kPi * x[0]) / (4.0 * kPi) + std::cos(2.0 * kPi * x[1]) / (2.0 * kPi));
      }, b1f, b2f, b3f);
      finish_cells(G, gamma, u, b1f, b2f, b3f, pgas);
      break;
    }
    case PMHD_PGEN_BLAST: {  // SURVEY.md §8d M3 (Athena++ mhd blast)
      const double xcen[3] = {0.5 * (cfg->mesh.xmin[0] + cfg->mesh.xmax[0]),
                              0.5 * (cfg->mesh.xmin[1] + cfg->mesh.xmax[1]),
                              0.5 * (cfg->mesh.xmin[2] + cfg->mesh.xmax[2])};
      for (int k = G.ks; k < G.ke; ++k)
        for (int j = G.js; j < G.je; ++j)
          for (int i = G.is; i < G.ie; ++i) {
            const double x = G.xc(0, c[0], i) - xcen[0], y = G.xc(1, c[1], j) - xcen[1];
            const double z = d3 ? G.xc(2, c[2], k) - xcen[2] : 0.0;
            const double r = std::sqrt(x * x + y * y + z * z);
            const size_t ci = G.cidx(k, j, i);
            u[ci] = cfg->blast_rho;
            u[nc + ci] = u[2 * nc + ci] = u[3 * nc + ci] = 0.0;
            pgas.push_back(r < cfg->blast_r ? cfg->blast_pin : cfg->blast_pout);
          }
      uniform_faces(G, cfg->blast_b, b1f, b2f, b3f);
      finish_cells(G, gamma, u, b1f, b2f, b3f, pgas);
      break;
    }
    case PMHD_PGEN_TURBULENCE: {  // SURVEY.md §8d M5 (decaying, no forcing)
      double scale = 1.0;
      const std::vector<TurbMode> modes = turb_modes(*cfg, &scale);
      double L[3];
      for (int a = 0; a < 3; ++a) L[a] = cfg->mesh.xmax[a] - cfg->mesh.xmin[a];
      const double d0 = cfg->uniform_w[0];
      for (int k = G.ks; k < G.ke; ++k)
        for (int j = G.js; j < G.je; ++j)
          for (int i = G.is; i < G.ie; ++i) {
            const double x = G.xc(0, c[0], i), y = G.xc(1, c[1], j), z = d3 ? G.xc(2, c[2], k) : 0.0;
            double v[3] = {0.0, 0.0, 0.0};
            for (const auto& m : modes) {
              const double ph = 2.0 * kPi * (m.k[0] * x / L[0] + m.k[1] * y / L[1] + m.k[2] * z / L[2]) + m.phase;
              const double s = std::sin(ph);
              for (int a = 0; a < 3; ++a) v[a] += m.a[a] * s;
            }
            const size_t ci = G.cidx(k, j, i);
            u[ci] = d0;
            for (int a = 0; a < 3; ++a) u[(1 + a) * nc + ci] = d0 * scale * v[a];
            pgas.push_back(cfg->uniform_w[4]);
          }
      uniform_faces(G, cfg->uniform_w + 5, b1f, b2f, b3f);
      finish_cells(G, gamma, u, b1f, b2f, b3f, pgas);
      break;
    }
    case PMHD_PGEN_UNIFORM: {
      const double* w = cfg->uniform_w;
      for (int k = G.ks; k < G.ke; ++k)
        for (int j = G.js; j < G.je; ++j)
          for (int i = G.is; i < G.ie; ++i) {
            const size_t ci = G.cidx(k, j, i);
            u[ci] = w[0];
            for (int a = 0; a < 3; ++a) u[(1 + a) * nc + ci] = w[0] * w[1 + a];
            pgas.push_back(w[4]);
          }
      uniform_faces(G, w + 5, b1f, b2f, b3f);
      finish_cells(G, gamma, u, b1f, b2f, b3f, pgas);
      break;
    }
    default:
      return PMHD_ERR_CONFIG;
  }
  (void)g_dummy;
  return PMHD_OK;
}

int pmhd_host_exact_block(const pmhd_run_config* cfg, int gid, double t, double* u) {
  if (cfg->pgen != PMHD_PGEN_LINEAR_WAVE) return PMHD_ERR_UNSUPPORTED;
  const Geom G(cfg->mesh);
  int c[3];
  G.coords(gid, c);
  WaveEigen W;
  if (wave_eigen(*cfg, W)) return PMHD_ERR_CONFIG;
  const size_t nc = G.ncell();
  const double om = W.lambda * W.kmag;
  const bool d3 = G.dim == 3;
  for (int k = G.ks; k < G.ke; ++k)
    for (int j = G.js; j < G.je; ++j)
      for (int i = G.is; i < G.ie; ++i) {
        const double x = G.xc(0, c[0], i), y = G.xc(1, c[1], j), z = d3 ? G.xc(2, c[2], k) : 0.0;
        double q[8];
        wave_state(*cfg, W, W.k[0] * x + W.k[1] * y + W.k[2] * z - om * t, q);
        for (int v = 0; v < 8; ++v) u[v * nc + G.cidx(k, j, i)] = q[v];
      }
  return PMHD_OK;
}

}  // extern "C"
