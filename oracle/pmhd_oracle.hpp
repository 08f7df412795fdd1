// oracle/pmhd_oracle.hpp -- TEST INFRASTRUCTURE, not product code.
//
// CPU restatement of the reference's hot path: the K-Athena / Athena++
// second-order MHD update (VL2 predictor-corrector + PLM + HLLD/HLLE +
// constrained transport + conserved update + cons->prim), fp64.
//
// In the reference this path exists only as specification, so this file IS
// the executable definition that the CUDA path must reproduce bit for bit
// (parity build, nvcc --fmad=false) or to 1e-11 (FMA build):
//   algorithm
//   mhd_solver module
//   core_mesh module
//   layout / errors      /root/reference/proj/include/pmhd/defs.hpp:14-78,
//                        /root/reference/proj/include/pmhd/array.hpp:19-80
//   no FP contraction    /root/reference/proj/CMakeLists.txt:11-14
// HLLD, floors and the contact-upwind CT weights are not in the reference
// (HLLD is a SPEC non-goal; north_star requires it); they follow
// Miyoshi & Kusano (2005) and Gardiner & Stone (2005) as restated in
// DESIGN.md "Algorithm definition".  Those pieces are PARITY UNPINNED by any
// reference artefact: they are checked by SPEC properties (consistency,
// conservation, div B, convergence) and an independent textbook HLLD in tests.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
// this code.  The product path never links it.
#ifndef ORACLE_PMHD_ORACLE_HPP_
#define ORACLE_PMHD_ORACLE_HPP_

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <type_traits>
#include <string>
#include <vector>

#include "counting.hpp"
#include "pmhd_gpu.h"  // only for pmhd_mesh_desc / enums (plain C structs)

#ifdef ORACLE_USE_REF_EXEC
#include "pmhd/exec/dispatch.hpp"  // the reference's own par_for (dispatch.hpp:109-118)
#endif

namespace oracle {

// Variable indices: defs.hpp:22-25.
enum { IDN = 0, IM1 = 1, IM2 = 2, IM3 = 3, IEN = 4, IB1 = 5, IB2 = 6, IB3 = 7 };
enum { IV1 = 1, IV2 = 2, IV3 = 3, IPR = 4 };
constexpr int NCONS = 8, NHYDRO = 5, NWAVE = 7;  // defs.hpp:27-29

// HLLD degeneracy threshold (Miyoshi & Kusano 2005 / Athena++ SMALL_NUMBER).
constexpr double kSmall = 1.0e-8;

struct UnphysicalState : std::runtime_error {  // defs.hpp:51-62
  int stage, k, j, i;
  UnphysicalState(int s, int kk, int jj, int ii)
      : std::runtime_error("unphysical state"), stage(s), k(kk), j(jj), i(ii) {}
};
struct ConfigErr : std::runtime_error {  // defs.hpp:36-39
  using std::runtime_error::runtime_error;
};

//----------------------------------------------------------------------------
// Execution: par_for restated.  Pure maps: any split gives bitwise-identical
// arrays (dispatch.hpp:8-15).  Default = static contiguous chunks over k
// (SimdNested, dispatch.hpp:30-41) on a small fork/join pool;
// ORACLE_USE_REF_EXEC runs the reference's own par_for / ThreadPool instead.
struct Bounds { int ks, ke, js, je, is, ie; };
inline int g_workers = 1;

// Minimal persistent fork/join pool: job(w) for w in [0, n), caller is w = 0,
// returns after all workers finish (the par_for synchronization point,
// dispatch.hpp:106-108).
class Pool {
 public:
  static Pool& get() { static Pool p; return p; }
  void run(int n, const std::function<void(int)>& job) {
    if (n <= 1) { job(0); return; }
    {
      std::unique_lock<std::mutex> lk(mu_);
      while ((int)th_.size() < n - 1) {
        const int id = (int)th_.size() + 1;
        th_.emplace_back([this, id] { loop(id); });
      }
      job_ = &job; active_ = n - 1; left_ = n - 1; ++gen_;
    }
    cv_go_.notify_all();
    job(0);
    std::unique_lock<std::mutex> lk(mu_);
    cv_done_.wait(lk, [&] { return left_ == 0; });
    job_ = nullptr;
  }
  ~Pool() {
    { std::unique_lock<std::mutex> lk(mu_); stop_ = true; }
    cv_go_.notify_all();
    for (auto& t : th_) t.join();
  }

 private:
  void loop(int id) {
    long seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_go_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (id > active_) continue;
        job = job_;
      }
      (*job)(id);
      std::unique_lock<std::mutex> lk(mu_);
      if (--left_ == 0) cv_done_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_go_, cv_done_;
  const std::function<void(int)>* job_ = nullptr;
  long gen_ = 0;
  int active_ = 0, left_ = 0;
  bool stop_ = false;
};

template <class F>
inline void par3(const Bounds& b, F&& f) {
  if (b.ke <= b.ks || b.je <= b.js || b.ie <= b.is) return;
#ifdef ORACLE_USE_REF_EXEC
  pmhd::LoopPolicy pol;
  pol.pattern = pmhd::LoopPattern::SimdNested;
  pol.workers = g_workers;
  pmhd::LoopBounds lb;
  lb.ks = b.ks; lb.ke = b.ke; lb.js = b.js; lb.je = b.je; lb.is = b.is; lb.ie = b.ie;
  pmhd::par_for(pol, lb, f);
#else
  const int nk = b.ke - b.ks;
  const int nw = std::max(1, std::min(g_workers, nk));
  auto body = [&](int w) {
    const int chunk = (nk + nw - 1) / nw;  // static contiguous chunks over k
    const int k0 = b.ks + std::min(nk, chunk * w), k1 = b.ks + std::min(nk, chunk * (w + 1));
    for (int k = k0; k < k1; ++k)
      for (int j = b.js; j < b.je; ++j)
        for (int i = b.is; i < b.ie; ++i) f(k, j, i);
  };
  if (nw == 1) body(0);
  else Pool::get().run(nw, body);
#endif
}

//----------------------------------------------------------------------------
// Dense k-j-i array (array.hpp:19-48 semantics, i fastest).
template <class R>
struct Field {
  int n3 = 0, n2 = 0, n1 = 0;
  std::vector<R> a;
  void resize(int k, int j, int i) { n3 = k; n2 = j; n1 = i; a.assign(size_t(k) * j * i, R(0.0)); }
  R& operator()(int k, int j, int i) { return a[(size_t(k) * n2 + j) * n1 + i]; }
  const R& operator()(int k, int j, int i) const { return a[(size_t(k) * n2 + j) * n1 + i]; }
};

//----------------------------------------------------------------------------
// Physical constants of one run.
struct Phys {
  double gamma, gm1, igm1;
  int riemann, limiter, eos_mode, emf_mode;
  double dfloor, pfloor;
  explicit Phys(const pmhd_mesh_desc& d)
      : gamma(d.gamma), gm1(d.gamma - 1.0), igm1(1.0 / (d.gamma - 1.0)), riemann(d.riemann),
        limiter(d.limiter), eos_mode(d.eos_mode), emf_mode(d.emf_mode), dfloor(d.dfloor),
        pfloor(d.pfloor) {}
};

//============================================================================
// Pointwise physics.  The operation order written here is the definition the
// CUDA kernels mirror.

// prim_to_cons: E = p/(g-1) + rho v^2/2 + B^2/2, m = rho v.
template <class R>
inline void prim_to_cons(const R* w, const Phys& ph, R* u) {
  u[IDN] = w[IDN];
  u[IM1] = w[IDN] * w[IV1];
  u[IM2] = w[IDN] * w[IV2];
  u[IM3] = w[IDN] * w[IV3];
  const R ke = 0.5 * (u[IM1] * w[IV1] + u[IM2] * w[IV2] + u[IM3] * w[IV3]);
  const R pb = 0.5 * (w[IB1] * w[IB1] + w[IB2] * w[IB2] + w[IB3] * w[IB3]);
  u[IEN] = w[IPR] * ph.igm1 + ke + pb;
  u[IB1] = w[IB1]; u[IB2] = w[IB2]; u[IB3] = w[IB3];
}

// cons_to_prim.  u: 5 hydro vars (may be modified by floors
// when fix_u), b: cell-centred field.  Returns a bitmask: 1 = rho floored,
// 2 = p floored, 4 = unphysical (error mode: rho<=0 or p<=0).
template <class R>
inline int cons_to_prim(R* u, const R* b, const Phys& ph, R* w, bool fix_u) {
  int flags = 0;
  R d = u[IDN];
  if (ph.eos_mode == PMHD_EOS_FLOOR) {
    if (d < ph.dfloor) { d = ph.dfloor; flags |= 1; if (fix_u) u[IDN] = d; }
  } else if (!(d > 0.0)) {
    flags |= 4;
    d = 1.0;  // keep the arithmetic finite; the caller raises
  }
  const R id = 1.0 / d;
  const R v1 = u[IM1] * id, v2 = u[IM2] * id, v3 = u[IM3] * id;
  const R ke = 0.5 * (u[IM1] * v1 + u[IM2] * v2 + u[IM3] * v3);
  const R pb = 0.5 * (b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
  R p = ph.gm1 * (u[IEN] - ke - pb);
  if (ph.eos_mode == PMHD_EOS_FLOOR) {
    if (p < ph.pfloor) {
      p = ph.pfloor; flags |= 2;
      if (fix_u) u[IEN] = p * ph.igm1 + ke + pb;
    }
  } else if (!(p > 0.0)) {
    flags |= 4;
  }
  w[IDN] = d; w[IV1] = v1; w[IV2] = v2; w[IV3] = v3; w[IPR] = p;
  w[IB1] = b[0]; w[IB2] = b[1]; w[IB3] = b[2];
  return flags;
}

// fast_speed along the normal n of a rotated state,
// in the cancellation-free form c_f^2 = (q + sqrt(t^2 + 4 a^2 ct^2))/2,
// q = a^2+cax^2+ct^2, t = cax^2+ct^2-a^2 (algebraically equal to the SPEC form).
template <class R>
inline R fast_speed_n(R d, R p, R bn, R bt1, R bt2, double gamma) {
  using std::sqrt;
  const R id = 1.0 / d;
  const R asq = gamma * p * id;
  const R cax2 = bn * bn * id;
  const R ct2 = (bt1 * bt1 + bt2 * bt2) * id;
  const R qsq = cax2 + ct2 + asq;
  const R tmp = cax2 + ct2 - asq;
  return sqrt(0.5 * (qsq + sqrt(tmp * tmp + 4.0 * asq * ct2)));
}

// Rotated 7-state: d, vn, vt1, vt2, p, bt1, bt2 (Appendix A.3 of SURVEY.md).
// Lab indices of (vn,vt1,vt2) and (bt1,bt2) per direction.
inline void rot_indices(int dir, int iv[3], int ib[2]) {
  if (dir == 0) { iv[0] = IV1; iv[1] = IV2; iv[2] = IV3; ib[0] = IB2; ib[1] = IB3; }
  else if (dir == 1) { iv[0] = IV2; iv[1] = IV3; iv[2] = IV1; ib[0] = IB3; ib[1] = IB1; }
  else { iv[0] = IV3; iv[1] = IV1; iv[2] = IV2; ib[0] = IB1; ib[1] = IB2; }
}

// Physical 1-D flux and conserved state of a rotated state.
template <class R>
struct SideState {
  R u[7];  // d, mn, mt1, mt2, e, bt1, bt2
  R f[7];  // fluxes of the above
  R pt, vb, cf;
};

template <class R>
inline void side_state(const R* w, R bx, R bxsq, const Phys& ph, SideState<R>& s) {
  const R d = w[0], vx = w[1], vy = w[2], vz = w[3], p = w[4], by = w[5], bz = w[6];
  const R pb = 0.5 * (bxsq + by * by + bz * bz);
  s.pt = p + pb;
  s.u[0] = d;
  s.u[1] = d * vx;
  s.u[2] = d * vy;
  s.u[3] = d * vz;
  s.u[4] = p * ph.igm1 + 0.5 * (s.u[1] * vx + s.u[2] * vy + s.u[3] * vz) + pb;
  s.u[5] = by;
  s.u[6] = bz;
  s.vb = vx * bx + vy * by + vz * bz;
  s.f[0] = s.u[1];
  s.f[1] = s.u[1] * vx + s.pt - bxsq;
  s.f[2] = s.u[2] * vx - bx * by;
  s.f[3] = s.u[3] * vx - bx * bz;
  s.f[4] = (s.u[4] + s.pt) * vx - bx * s.vb;
  s.f[5] = by * vx - bx * vy;
  s.f[6] = bz * vx - bx * vz;
  s.cf = fast_speed_n(d, p, bx, by, bz, ph.gamma);
}

// HLLE with Davis bounds (D8).  Written so that F(W,W) = F(W)
// and the supersonic branches return F(U_L) / F(U_R) exactly.
template <class R>
inline void riemann_hlle(const R* wl, const R* wr, R bx, const Phys& ph, R* flx) {
  using std::fmin; using std::fmax;
  const R bxsq = bx * bx;
  SideState<R> L, Rt;
  side_state(wl, bx, bxsq, ph, L);
  side_state(wr, bx, bxsq, ph, Rt);
  const R sl = fmin(wl[1] - L.cf, wr[1] - Rt.cf);
  const R sr = fmax(wl[1] + L.cf, wr[1] + Rt.cf);
  if (sl >= 0.0) { for (int n = 0; n < 7; ++n) flx[n] = L.f[n]; return; }
  if (sr <= 0.0) { for (int n = 0; n < 7; ++n) flx[n] = Rt.f[n]; return; }
  const R ibd = 1.0 / (sr - sl);
  const R hs = 0.5 * (sr + sl);
  const R pm = sr * sl;
  for (int n = 0; n < 7; ++n)
    flx[n] = 0.5 * (L.f[n] + Rt.f[n]) + (hs * (L.f[n] - Rt.f[n]) + pm * (Rt.u[n] - L.u[n])) * ibd;
}

// HLLD (Miyoshi & Kusano 2005, J. Comput. Phys. 208, 315), restated.  The
// wave-speed estimate is the Davis bound used for HLLE; the degenerate cases
// (Bx^2 ~ rho (S-u)(S-S_M), Bx -> 0) use the 1e-8 relative threshold.
template <class R>
struct StarState {
  R d, vy, vz, by, bz, e, vb;
};

template <class R>
inline void hlld_star(const R* w, const SideState<R>& S, R bx, R bxsq, R sm, R ptst, R sd,
                      R sdd, R sdm, StarState<R>& st) {
  using std::fabs;
  const R isdm = 1.0 / sdm;
  st.d = sdd * isdm;
  const R tmp = sdd * sdm - bxsq;
  if (fabs(tmp) < kSmall * ptst) {
    st.vy = w[2]; st.vz = w[3]; st.by = w[5]; st.bz = w[6];
  } else {
    const R itmp = 1.0 / tmp;
    const R mfact = bx * (sm - w[1]) * itmp;
    st.vy = w[2] - w[5] * mfact;
    st.vz = w[3] - w[6] * mfact;
    const R bfact = (sdd * sd - bxsq) * itmp;
    st.by = w[5] * bfact;
    st.bz = w[6] * bfact;
  }
  st.vb = sm * bx + st.vy * st.by + st.vz * st.bz;
  st.e = (sd * S.u[4] - S.pt * w[1] + ptst * sm + bx * (S.vb - st.vb)) * isdm;
}

template <class R>
inline void riemann_hlld(const R* wl, const R* wr, R bx, const Phys& ph, R* flx) {
  using std::fmin; using std::fmax; using std::fabs; using std::sqrt;
  const R bxsq = bx * bx;
  SideState<R> L, Rt;
  side_state(wl, bx, bxsq, ph, L);
  side_state(wr, bx, bxsq, ph, Rt);
  const R vxl = wl[1], vxr = wr[1];
  const R sl = fmin(vxl - L.cf, vxr - Rt.cf);
  const R sr = fmax(vxl + L.cf, vxr + Rt.cf);
  if (sl >= 0.0) { for (int n = 0; n < 7; ++n) flx[n] = L.f[n]; return; }
  if (sr <= 0.0) { for (int n = 0; n < 7; ++n) flx[n] = Rt.f[n]; return; }

  const R sdl = sl - vxl, sdr = sr - vxr;
  const R sdld = sdl * wl[0], sdrd = sdr * wr[0];
  const R idn = 1.0 / (sdrd - sdld);
  const R sm = (sdrd * vxr - sdld * vxl - Rt.pt + L.pt) * idn;               // M&K Eq. 38
  const R ptst = (sdrd * L.pt - sdld * Rt.pt + sdld * sdrd * (vxr - vxl)) * idn;  // Eq. 41
  const R sdml = sl - sm, sdmr = sr - sm;

  StarState<R> Ls, Rs;  // Eqs. 43-48
  hlld_star(wl, L, bx, bxsq, sm, ptst, sdl, sdld, sdml, Ls);
  hlld_star(wr, Rt, bx, bxsq, sm, ptst, sdr, sdrd, sdmr, Rs);

  const R sqdl = sqrt(Ls.d), sqdr = sqrt(Rs.d);
  const R abx = fabs(bx);
  const R slst = sm - abx / sqdl;  // Eq. 51
  const R srst = sm + abx / sqdr;

  R ul1[7], ur1[7];
  ul1[0] = Ls.d; ul1[1] = Ls.d * sm; ul1[2] = Ls.d * Ls.vy; ul1[3] = Ls.d * Ls.vz;
  ul1[4] = Ls.e; ul1[5] = Ls.by; ul1[6] = Ls.bz;
  ur1[0] = Rs.d; ur1[1] = Rs.d * sm; ur1[2] = Rs.d * Rs.vy; ur1[3] = Rs.d * Rs.vz;
  ur1[4] = Rs.e; ur1[5] = Rs.by; ur1[6] = Rs.bz;

  if (slst >= 0.0) {  // F*_L = F_L + S_L (U*_L - U_L)         Eq. 64
    for (int n = 0; n < 7; ++n) flx[n] = L.f[n] + sl * (ul1[n] - L.u[n]);
    return;
  }
  if (srst <= 0.0) {  // F*_R
    for (int n = 0; n < 7; ++n) flx[n] = Rt.f[n] + sr * (ur1[n] - Rt.u[n]);
    return;
  }
  // double-star states, Eqs. 59-63
  R ul2[7], ur2[7];
  if (0.5 * bxsq < kSmall * ptst) {
    for (int n = 0; n < 7; ++n) { ul2[n] = ul1[n]; ur2[n] = ur1[n]; }
  } else {
    using std::copysign;
    const R invsum = 1.0 / (sqdl + sqdr);
    const R sgn = copysign(R(1.0), bx);
    const R vy2 = (sqdl * Ls.vy + sqdr * Rs.vy + sgn * (Rs.by - Ls.by)) * invsum;
    const R vz2 = (sqdl * Ls.vz + sqdr * Rs.vz + sgn * (Rs.bz - Ls.bz)) * invsum;
    const R sq2 = sgn * sqdl * sqdr;
    const R by2 = (sqdl * Rs.by + sqdr * Ls.by + sq2 * (Rs.vy - Ls.vy)) * invsum;
    const R bz2 = (sqdl * Rs.bz + sqdr * Ls.bz + sq2 * (Rs.vz - Ls.vz)) * invsum;
    const R vb2 = sm * bx + vy2 * by2 + vz2 * bz2;
    ul2[0] = Ls.d; ul2[1] = ul1[1]; ul2[2] = Ls.d * vy2; ul2[3] = Ls.d * vz2;
    ul2[4] = Ls.e - sqdl * sgn * (Ls.vb - vb2); ul2[5] = by2; ul2[6] = bz2;
    ur2[0] = Rs.d; ur2[1] = ur1[1]; ur2[2] = Rs.d * vy2; ur2[3] = Rs.d * vz2;
    ur2[4] = Rs.e + sqdr * sgn * (Rs.vb - vb2); ur2[5] = by2; ur2[6] = bz2;
  }
  if (sm >= 0.0) {  // F**_L = F*_L + S*_L (U**_L - U*_L)        Eq. 65
    for (int n = 0; n < 7; ++n) {
      const R f1 = L.f[n] + sl * (ul1[n] - L.u[n]);
      flx[n] = f1 + slst * (ul2[n] - ul1[n]);
    }
  } else {
    for (int n = 0; n < 7; ++n) {
      const R f1 = Rt.f[n] + sr * (ur1[n] - Rt.u[n]);
      flx[n] = f1 + srst * (ur2[n] - ur1[n]);
    }
  }
}

// Roe flux (the paper's solver):
// F = (F_L + F_R)/2 - R|Lambda|L (U_R - U_L)/2 with the eigensystem of the
// flux Jacobian at the Roe state: rho = sqrt(rho_L rho_R), v and the total
// enthalpy density-weighted, transverse B weighted by the OTHER side's
// sqrt(rho), normal B = the face value.  The decomposition is done in
// primitive variables (rho, vn, vt1, vt2, p, bt1, bt2) linearised at the Roe
// state, with the Roe & Balsara (1996) eigenvector normalisation; B_t = 0 uses
// beta = (1,1)/sqrt 2, sgn(0) = +1.  Returns false (caller falls back to HLLE
// and counts it) when the Roe state has a^2 <= 0.
template <class R>
inline bool riemann_roe(const R* wl, const R* wr, R bx, const Phys& ph, R* flx) {
  using std::sqrt; using std::fabs; using std::fmax; using std::fmin;
  const R bxsq = bx * bx;
  SideState<R> L, Rt;
  side_state(wl, bx, bxsq, ph, L);
  side_state(wr, bx, bxsq, ph, Rt);
  const R sdl = sqrt(wl[0]), sdr = sqrt(wr[0]);
  const R isum = 1.0 / (sdl + sdr);
  const R d = sdl * sdr;
  const R u = (sdl * wl[1] + sdr * wr[1]) * isum;
  const R v = (sdl * wl[2] + sdr * wr[2]) * isum;
  const R w = (sdl * wl[3] + sdr * wr[3]) * isum;
  const R h = ((L.u[4] + L.pt) / sdl + (Rt.u[4] + Rt.pt) / sdr) * isum;  // Roe total enthalpy
  const R by = (sdr * wl[5] + sdl * wr[5]) * isum;
  const R bz = (sdr * wl[6] + sdl * wr[6]) * isum;
  const R id = 1.0 / d;
  const R vsq = u * u + v * v + w * w;
  const R btsq = by * by + bz * bz;
  const R asq = ph.gm1 * (h - 0.5 * vsq - (bxsq + btsq) * id);
  if (!(asq > 0.0)) return false;
  const R ca2 = bxsq * id, bt2 = btsq * id;
  const R tsum = ca2 + bt2 + asq, tdif = ca2 + bt2 - asq;
  const R cf2 = 0.5 * (tsum + sqrt(tdif * tdif + 4.0 * asq * bt2));
  const R cs2 = asq * ca2 / cf2;  // c_f^2 c_s^2 = a^2 c_a^2
  const R cf = sqrt(cf2), cs = sqrt(cs2), ca = sqrt(ca2), a = sqrt(asq);
  R af, as;
  const R dfs = cf2 - cs2;
  if (!(dfs > 0.0)) {
    af = 1.0; as = 0.0;
  } else {
    const R idfs = 1.0 / dfs;
    af = sqrt(fmax(R(0.0), fmin(R(1.0), (asq - cs2) * idfs)));
    as = sqrt(fmax(R(0.0), fmin(R(1.0), (cf2 - asq) * idfs)));
  }
  const R bt = sqrt(btsq);
  R bety, betz;
  if (bt > 0.0) {
    const R ibt = 1.0 / bt;
    bety = by * ibt; betz = bz * ibt;
  } else {
    bety = R(0.70710678118654752440); betz = R(0.70710678118654752440);
  }
  const R sgn = (bx >= 0.0) ? R(1.0) : R(-1.0);
  const R sd = sqrt(d);
  const R isd = 1.0 / sd;
  // dW = (dW/dU) dU at the Roe state
  R du[7];
  for (int n = 0; n < 7; ++n) du[n] = Rt.u[n] - L.u[n];
  const R dr = du[0];
  const R dvx = (du[1] - u * dr) * id, dvy = (du[2] - v * dr) * id, dvz = (du[3] - w * dr) * id;
  const R dby = du[5], dbz = du[6];
  const R dp = ph.gm1 * (du[4] - (u * du[1] + v * du[2] + w * du[3]) + 0.5 * vsq * dr -
                         (by * dby + bz * dbz));
  // wave amplitudes alpha_k = l_k . dW
  const R ia2 = 1.0 / asq;
  const R h2a = 0.5 * ia2;
  const R q = 0.5 * isd / a;
  const R dvt = bety * dvy + betz * dvz;
  const R dbt = bety * dby + betz * dbz;
  const R tfa = af * cf * h2a * dvx, tfs = as * cs * sgn * h2a * dvt;
  const R tfp = af * h2a * id * dp, tfb = as * q * dbt;
  const R am_f = tfp + tfb - tfa + tfs, ap_f = tfp + tfb + tfa - tfs;
  const R tav = 0.5 * (bety * dvz - betz * dvy);
  const R tab = 0.5 * sgn * isd * (betz * dby - bety * dbz);
  const R am_a = tav - tab, ap_a = tav + tab;
  const R tsa = as * cs * h2a * dvx, tss = af * cf * sgn * h2a * dvt;
  const R tsp = as * h2a * id * dp, tsb = af * q * dbt;
  const R am_s = tsp - tsb - tsa - tss, ap_s = tsp - tsb + tsa + tss;
  const R a_e = dr - dp * ia2;
  // |lambda_k| alpha_k
  const R wfm = fabs(u - cf) * am_f, wfp = fabs(u + cf) * ap_f;
  const R wam = fabs(u - ca) * am_a, wap = fabs(u + ca) * ap_a;
  const R wsm = fabs(u - cs) * am_s, wsp = fabs(u + cs) * ap_s;
  const R we = fabs(u) * a_e;
  // D_W = sum_k |lambda_k| alpha_k r_k (primitive right eigenvectors)
  const R sf = wfm + wfp, ss = wsm + wsp;
  const R Dr = d * (af * sf + as * ss) + we;
  const R Dvx = af * cf * (wfp - wfm) + as * cs * (wsp - wsm);
  const R tm = as * cs * sgn * (wfm - wfp) + af * cf * sgn * (wsp - wsm);
  const R Dvy = bety * tm - betz * (wam + wap);
  const R Dvz = betz * tm + bety * (wam + wap);
  const R Dp = d * asq * (af * sf + as * ss);
  const R tb = sd * a * (as * sf - af * ss);
  const R ta = sgn * sd * (wap - wam);
  const R Dby = bety * tb + betz * ta;
  const R Dbz = betz * tb - bety * ta;
  // D_U = (dU/dW) D_W
  R D[7];
  D[0] = Dr;
  D[1] = u * Dr + d * Dvx;
  D[2] = v * Dr + d * Dvy;
  D[3] = w * Dr + d * Dvz;
  D[4] = 0.5 * vsq * Dr + d * (u * Dvx + v * Dvy + w * Dvz) + Dp * ph.igm1 + by * Dby + bz * Dbz;
  D[5] = Dby;
  D[6] = Dbz;
  for (int n = 0; n < 7; ++n) flx[n] = 0.5 * (L.f[n] + Rt.f[n]) - 0.5 * D[n];
  return true;
}

// PLM slope: MC (monotonized central) or van Leer limiter,
// applied componentwise to primitives.  Zero at extrema; exact on linear data.
template <class R>
inline R plm_slope(R qm, R q0, R qp, int limiter) {
  using std::fmin; using std::fabs; using std::copysign;
  const R dql = q0 - qm, dqr = qp - q0;
  const R dq2 = dql * dqr;
  if (!(dq2 > 0.0)) return R(0.0);
  if (limiter == PMHD_LIMITER_MC) {
    const R dqc = 0.5 * (dql + dqr);
    const R lim = 2.0 * fmin(fabs(dql), fabs(dqr));
    return copysign(fmin(fabs(dqc), lim), dqc);
  }
  return 2.0 * dq2 / (dql + dqr);
}

// Riemann solve at one face + the CT by-products.  out: 5 hydro fluxes in the
// ROTATED order (d, mn, mt1, mt2, e), ey = -F(bt1), ez = F(bt2) (the face
// electric fields, E = -v x B, Athena++ convention), and the
// contact-upwind weight (1: upwind cell is the low side, 0: high side;
// Gardiner & Stone 2005 Eq. 50).  The weight is the continuous Athena++ form
// w = 1/2 + clamp(1024 (dt/dx) F_rho / (rho_L + rho_R), -1/2, 1/2) [ext]:
// a pure sign(F_rho) switch flips 0 <-> 1 on round-off noise of a vanishing
// mass flux and turns 1-ulp differences into O(dt dE) field differences.
// c1024 = 1024 * dt / dx_dir (full-cycle dt, both stages).
// Returns 1 when the Roe solver fell back to HLLE at this face.
template <class R>
inline int face_solve(const R* wl, const R* wr, R bx, const Phys& ph, double c1024, R* out) {
  using std::fmin; using std::fmax;
  R flx[7];
  int fb = 0;
  if (ph.riemann == PMHD_RIEMANN_HLLE) riemann_hlle(wl, wr, bx, ph, flx);
  else if (ph.riemann == PMHD_RIEMANN_ROE) {
    if (!riemann_roe(wl, wr, bx, ph, flx)) { riemann_hlle(wl, wr, bx, ph, flx); fb = 1; }
  } else riemann_hlld(wl, wr, bx, ph, flx);
  for (int n = 0; n < 5; ++n) out[n] = flx[n];
  out[5] = -flx[5];
  out[6] = flx[6];
  const R vc = c1024 * flx[0] / (wl[0] + wr[0]);
  out[7] = 0.5 + fmax(R(-0.5), fmin(R(0.5), vc));
  return fb;
}

//============================================================================
// Mesh / MeshBlock and the VL2 update.

struct Geometry {
  int nx[3], mb[3], nb[3], ng, dim;
  int n[3];            // block array extents incl. ghosts (n1,n2,n3)
  int is, ie, js, je, ks, ke;
  double dx[3], xmin[3], xmax[3];
  int nblocks;
  explicit Geometry(const pmhd_mesh_desc& d) {
    if (d.ng < 2) throw ConfigErr("ng must be >= 2");
    for (int a = 0; a < 3; ++a) {
      if (d.nx[a] < 1 || d.mb[a] < 1) throw ConfigErr("cell counts must be positive");
      if (d.nx[a] % d.mb[a] != 0) throw ConfigErr("global cells not divisible by meshblock cells");
      if (!(d.xmax[a] > d.xmin[a])) throw ConfigErr("empty domain extent");
    }
    if (d.nx[1] == 1) throw ConfigErr("1D meshes are not supported");
    if (d.mb[0] <= d.ng || d.mb[1] <= d.ng || (d.nx[2] > 1 && d.mb[2] <= d.ng))
      throw ConfigErr("meshblock must have more than ng cells per dimension");
    if (!(d.gamma > 1.0)) throw ConfigErr("gamma must be > 1");
    if (!(d.cfl > 0.0 && d.cfl < 1.0)) throw ConfigErr("cfl must be in (0,1)");
    dim = (d.nx[2] == 1) ? 2 : 3;
    ng = d.ng;
    nblocks = 1;
    for (int a = 0; a < 3; ++a) {
      nx[a] = d.nx[a]; mb[a] = d.mb[a]; nb[a] = d.nx[a] / d.mb[a]; nblocks *= nb[a];
      xmin[a] = d.xmin[a]; xmax[a] = d.xmax[a];
      dx[a] = (d.xmax[a] - d.xmin[a]) / d.nx[a];
      const int g = (a == 2 && dim == 2) ? 0 : ng;
      n[a] = mb[a] + 2 * g;
    }
    is = ng; ie = ng + mb[0]; js = ng; je = ng + mb[1];
    if (dim == 3) { ks = ng; ke = ng + mb[2]; } else { ks = 0; ke = 1; }
  }
  void block_coords(int gid, int c[3]) const {
    c[0] = gid % nb[0]; c[1] = (gid / nb[0]) % nb[1]; c[2] = gid / (nb[0] * nb[1]);
  }
  int gid_of(const int c[3]) const {
    return (((c[2] + nb[2]) % nb[2]) * nb[1] + ((c[1] + nb[1]) % nb[1])) * nb[0] +
           ((c[0] + nb[0]) % nb[0]);
  }
};

template <class R>
struct State {
  Field<R> u[NHYDRO];  // hydro conserved (Bcc is derived from the faces)
  Field<R> b1, b2, b3;  // face fields
  void alloc(const Geometry& g) {
    for (auto& f : u) f.resize(g.n[2], g.n[1], g.n[0]);
    b1.resize(g.n[2], g.n[1], g.n[0] + 1);
    b2.resize(g.n[2], g.n[1] + 1, g.n[0]);
    b3.resize(g.n[2] + 1, g.n[1], g.n[0]);
  }
};

template <class R>
struct Block {
  int gid, c[3];
  State<R> A, B;       // A = u^n (and u^{n+1}), B = u^{n+1/2}
  Field<R> w[NCONS];   // stage-input primitives incl. Bcc (all cells)
  Field<R> wend[NCONS];  // end-of-stage primitives (active cells)
  Field<R> fx[3][8];   // face data per direction
  Field<R> e1, e2, e3;  // corner EMFs
};

template <class R>
class Mesh {
 public:
  Geometry g;
  Phys ph;
  double cfl;
  std::vector<Block<R>> blocks;      // the blocks this rank owns, in gid order
  std::vector<int> local_of;         // gid -> index in blocks, -1 if remote
  long long floor_count = 0;
  std::atomic<long long> fallbacks{0};  // Roe -> HLLE fallbacks since reset

  // gids: the blocks this rank owns (all blocks when empty).
  explicit Mesh(const pmhd_mesh_desc& d, std::vector<int> gids = {}) : g(d), ph(d), cfl(d.cfl) {
    if (gids.empty())
      for (int b = 0; b < g.nblocks; ++b) gids.push_back(b);
    std::sort(gids.begin(), gids.end());
    local_of.assign(g.nblocks, -1);
    blocks.resize(gids.size());
    for (size_t lb = 0; lb < gids.size(); ++lb) {
      if (gids[lb] < 0 || gids[lb] >= g.nblocks) throw ConfigErr("gid out of range");
      local_of[gids[lb]] = int(lb);
      Block<R>& B = blocks[lb];
      B.gid = gids[lb];
      g.block_coords(B.gid, B.c);
      B.A.alloc(g); B.B.alloc(g);
      for (auto& f : B.w) f.resize(g.n[2], g.n[1], g.n[0]);
      for (auto& f : B.wend) f.resize(g.n[2], g.n[1], g.n[0]);
      for (int v = 0; v < 8; ++v) {
        B.fx[0][v].resize(g.n[2], g.n[1], g.n[0] + 1);
        B.fx[1][v].resize(g.n[2], g.n[1] + 1, g.n[0]);
        B.fx[2][v].resize(g.n[2] + 1, g.n[1], g.n[0]);
      }
      B.e1.resize(g.n[2] + 1, g.n[1] + 1, g.n[0]);
      B.e2.resize(g.n[2] + 1, g.n[1], g.n[0] + 1);
      B.e3.resize(g.n[2], g.n[1] + 1, g.n[0] + 1);
    }
  }

  Bounds all_cells() const { return Bounds{0, g.n[2], 0, g.n[1], 0, g.n[0]}; }
  Bounds active() const { return Bounds{g.ks, g.ke, g.js, g.je, g.is, g.ie}; }

  // face_to_center_b
  static void bcc(const State<R>& S, int k, int j, int i, R* b) {
    b[0] = 0.5 * (S.b1(k, j, i) + S.b1(k, j, i + 1));
    b[1] = 0.5 * (S.b2(k, j, i) + S.b2(k, j + 1, i));
    b[2] = 0.5 * (S.b3(k, j, i) + S.b3(k + 1, j, i));
  }

  // Global active coordinates of a local cell (for UnphysicalStateError).
  void global_cell(const Block<R>& B, int k, int j, int i, int out[3]) const {
    out[0] = B.c[0] * g.mb[0] + (i - g.is);
    out[1] = B.c[1] * g.mb[1] + (j - g.js);
    out[2] = (g.dim == 3) ? B.c[2] * g.mb[2] + (k - g.ks) : 0;
  }

  // Stage-input cons->prim over all cells (floors applied to w only, not
  // counted; error mode reports).  Definition: DESIGN.md "floors".
  void c2p_all(Block<R>& B, const State<R>& S, std::atomic<long long>* bad) {
    par3(all_cells(), [&](int k, int j, int i) {
      R u[NHYDRO], b[3], w[NCONS];
      for (int v = 0; v < NHYDRO; ++v) u[v] = S.u[v](k, j, i);
      bcc(S, k, j, i, b);
      const int fl = cons_to_prim(u, b, ph, w, false);
      for (int v = 0; v < NCONS; ++v) B.w[v](k, j, i) = w[v];
      if ((fl & 4) && k >= g.ks && k < g.ke && j >= g.js && j < g.je && i >= g.is && i < g.ie)
        record_bad(B, k, j, i, bad);  // ghosts are images of active cells
    });
  }

  void record_bad(const Block<R>& B, int k, int j, int i, std::atomic<long long>* bad) {
    int gc[3];
    global_cell(B, k, j, i, gc);
    const long long key = ((long long)gc[2] * g.nx[1] + gc[1]) * g.nx[0] + gc[0];
    long long cur = bad->load();
    while (key < cur && !bad->compare_exchange_weak(cur, key)) {}
  }

  // Riemann fluxes in direction dir over the face range needed by CT
  // (SURVEY.md Appendix A.2): normal faces [s, e], transverse extended by one
  // cell on each side (by one layer in x3 only in 3D).
  void fluxes(Block<R>& B, const State<R>& in, int dir, bool plm, double dt) {
    int iv[3], ib[2];
    rot_indices(dir, iv, ib);
    const double c1024 = 1024.0 * dt / g.dx[dir];
    const int d3 = (g.dim == 3) ? 1 : 0;
    Bounds fb;
    if (dir == 0) fb = Bounds{g.ks - d3, g.ke + d3, g.js - 1, g.je + 1, g.is, g.ie + 1};
    else if (dir == 1) fb = Bounds{g.ks - d3, g.ke + d3, g.js, g.je + 1, g.is - 1, g.ie + 1};
    else fb = Bounds{g.ks, g.ke + 1, g.js - 1, g.je + 1, g.is - 1, g.ie + 1};
    const int di = (dir == 0), dj = (dir == 1), dk = (dir == 2);
    const Field<R>& bn = (dir == 0) ? in.b1 : (dir == 1 ? in.b2 : in.b3);
    const int vars[7] = {IDN, iv[0], iv[1], iv[2], IPR, ib[0], ib[1]};
    par3(fb, [&](int k, int j, int i) {
      R wl[7], wr[7];
      constexpr bool counting = std::is_same<R, Counting>::value;
      const double r0 = counting ? g_tally.total() : 0.0;
      for (int n = 0; n < 7; ++n) {
        const Field<R>& q = B.w[vars[n]];
        const R qm1 = q(k - dk, j - dj, i - di);  // cell on the low side
        const R q0 = q(k, j, i);                  // cell on the high side
        if (plm) {
          const R qm2 = q(k - 2 * dk, j - 2 * dj, i - 2 * di);
          const R qp1 = q(k + dk, j + dj, i + di);
          wl[n] = qm1 + 0.5 * plm_slope(qm2, qm1, q0, ph.limiter);
          wr[n] = q0 - 0.5 * plm_slope(qm1, q0, qp1, ph.limiter);
        } else {  // donor cell (stage 1)
          wl[n] = qm1;
          wr[n] = q0;
        }
      }
      R out[8];
      const double r1 = counting ? g_tally.total() : 0.0;
      if (face_solve(wl, wr, bn(k, j, i), ph, c1024, out)) fallbacks.fetch_add(1);
      if (counting) {  // counting meshes run one worker
        g_region[1] += r1 - r0;
        g_region[2] += g_tally.total() - r1;
      }
      B.fx[dir][IDN](k, j, i) = out[0];  // un-rotate momentum fluxes
      B.fx[dir][iv[0]](k, j, i) = out[1];
      B.fx[dir][iv[1]](k, j, i) = out[2];
      B.fx[dir][iv[2]](k, j, i) = out[3];
      B.fx[dir][IEN](k, j, i) = out[4];
      B.fx[dir][5](k, j, i) = out[5];
      B.fx[dir][6](k, j, i) = out[6];
      B.fx[dir][7](k, j, i) = out[7];
    });
  }

  // Cell-centred E = -v x B of the stage-input state.
  static R ecc(const Block<R>& B, int comp, int k, int j, int i) {
    const R v1 = B.w[IV1](k, j, i), v2 = B.w[IV2](k, j, i), v3 = B.w[IV3](k, j, i);
    const R b1 = B.w[IB1](k, j, i), b2 = B.w[IB2](k, j, i), b3 = B.w[IB3](k, j, i);
    if (comp == 0) return v3 * b2 - v2 * b3;
    if (comp == 1) return v1 * b3 - v3 * b1;
    return v2 * b1 - v1 * b2;
  }

  // Gardiner & Stone (2005) contact-upwind corner EMF in the (a,b) plane.
  // ea_b / ea_bm: E on the a-faces adjacent to the corner at b and b-1;
  // eb_a / eb_am: E on the b-faces at a and a-1; w*: their upwind weights;
  // c_ab..: cell-centred E of the four cells around the corner.
  static R corner_emf(int mode, R ea_b, R ea_bm, R eb_a, R eb_am, R wa_b, R wa_bm, R wb_a,
                      R wb_am, R c_ab, R c_amb, R c_abm, R c_ambm) {
    if (mode == PMHD_EMF_ARITH) return 0.25 * ((ea_b + ea_bm) + (eb_a + eb_am));
    // GS05 Eq. 41: avg(faces) + dy/8 [(dE/dy)_{j-3/4} - (dE/dy)_{j-1/4}] + dx/8 [...]
    // = avg(faces) + 1/4 sum of upwinded (E_face - E_cell): exact for E
    // quadratic along each axis (Athena++ calculate_corner_e has the same form).
    const R t0 = ea_b + ea_bm;
    const R t1 = eb_a + eb_am;
    const R t2 = wa_b * (eb_am - c_amb) + (1.0 - wa_b) * (eb_a - c_ab);
    const R t3 = wa_bm * (eb_am - c_ambm) + (1.0 - wa_bm) * (eb_a - c_abm);
    const R t4 = wb_a * (ea_bm - c_abm) + (1.0 - wb_a) * (ea_b - c_ab);
    const R t5 = wb_am * (ea_bm - c_ambm) + (1.0 - wb_am) * (ea_b - c_amb);
    return 0.25 * (t0 + t1 + t2 + t3 + t4 + t5);
  }

  void emfs(Block<R>& B) {
    const int mode = ph.emf_mode;
    auto& X1 = B.fx[0]; auto& X2 = B.fx[1]; auto& X3 = B.fx[2];
    // E3 at (x_{i-1/2}, y_{j-1/2}, z_k): a = x1 faces, b = x2 faces.
    par3(Bounds{g.ks, g.ke, g.js, g.je + 1, g.is, g.ie + 1}, [&](int k, int j, int i) {
      B.e3(k, j, i) = corner_emf(mode, X1[5](k, j, i), X1[5](k, j - 1, i), X2[6](k, j, i),
                                 X2[6](k, j, i - 1), X1[7](k, j, i), X1[7](k, j - 1, i),
                                 X2[7](k, j, i), X2[7](k, j, i - 1), ecc(B, 2, k, j, i),
                                 ecc(B, 2, k, j, i - 1), ecc(B, 2, k, j - 1, i),
                                 ecc(B, 2, k, j - 1, i - 1));
    });
    if (g.dim == 3) {
      // E1 at (x_i, y_{j-1/2}, z_{k-1/2}): a = x2 faces, b = x3 faces.
      par3(Bounds{g.ks, g.ke + 1, g.js, g.je + 1, g.is, g.ie}, [&](int k, int j, int i) {
        B.e1(k, j, i) = corner_emf(mode, X2[5](k, j, i), X2[5](k - 1, j, i), X3[6](k, j, i),
                                   X3[6](k, j - 1, i), X2[7](k, j, i), X2[7](k - 1, j, i),
                                   X3[7](k, j, i), X3[7](k, j - 1, i), ecc(B, 0, k, j, i),
                                   ecc(B, 0, k, j - 1, i), ecc(B, 0, k - 1, j, i),
                                   ecc(B, 0, k - 1, j - 1, i));
      });
      // E2 at (x_{i-1/2}, y_j, z_{k-1/2}): a = x3 faces, b = x1 faces.
      par3(Bounds{g.ks, g.ke + 1, g.js, g.je, g.is, g.ie + 1}, [&](int k, int j, int i) {
        B.e2(k, j, i) = corner_emf(mode, X3[5](k, j, i), X3[5](k, j, i - 1), X1[6](k, j, i),
                                   X1[6](k - 1, j, i), X3[7](k, j, i), X3[7](k, j, i - 1),
                                   X1[7](k, j, i), X1[7](k - 1, j, i), ecc(B, 1, k, j, i),
                                   ecc(B, 1, k - 1, j, i), ecc(B, 1, k, j, i - 1),
                                   ecc(B, 1, k - 1, j, i - 1));
      });
    } else {
      // 2D: E1, E2 are uniform in x3 and equal the single face value.
      par3(Bounds{0, 1, g.js, g.je + 1, g.is, g.ie}, [&](int k, int j, int i) {
        B.e1(0, j, i) = X2[5](0, j, i);
        B.e1(1, j, i) = X2[5](0, j, i);
        (void)k;
      });
      par3(Bounds{0, 1, g.js, g.je, g.is, g.ie + 1}, [&](int k, int j, int i) {
        B.e2(0, j, i) = X1[6](0, j, i);
        B.e2(1, j, i) = X1[6](0, j, i);
        (void)k;
      });
    }
  }

  // Conserved + CT update, then end-of-stage cons->prim of active cells.
  void update(Block<R>& B, const State<R>& base, State<R>& out, double beta, double dt,
              std::atomic<long long>* bad, std::atomic<long long>* nfloor) {
    const double bdt = beta * dt;
    const double c1 = bdt / g.dx[0], c2 = bdt / g.dx[1], c3 = bdt / g.dx[2];
    auto& X1 = B.fx[0]; auto& X2 = B.fx[1]; auto& X3 = B.fx[2];
    const bool d3 = (g.dim == 3);
    par3(active(), [&](int k, int j, int i) {
      for (int v = 0; v < NHYDRO; ++v) {
        R du = c1 * (X1[v](k, j, i + 1) - X1[v](k, j, i)) + c2 * (X2[v](k, j + 1, i) - X2[v](k, j, i));
        if (d3) du = du + c3 * (X3[v](k + 1, j, i) - X3[v](k, j, i));
        out.u[v](k, j, i) = base.u[v](k, j, i) - du;
      }
    });
    // b1f on faces i in [is, ie]
    par3(Bounds{g.ks, g.ke, g.js, g.je, g.is, g.ie + 1}, [&](int k, int j, int i) {
      if (d3)
        out.b1(k, j, i) = base.b1(k, j, i) - (c2 * (B.e3(k, j + 1, i) - B.e3(k, j, i)) -
                                              c3 * (B.e2(k + 1, j, i) - B.e2(k, j, i)));
      else
        out.b1(k, j, i) = base.b1(k, j, i) - c2 * (B.e3(k, j + 1, i) - B.e3(k, j, i));
    });
    par3(Bounds{g.ks, g.ke, g.js, g.je + 1, g.is, g.ie}, [&](int k, int j, int i) {
      if (d3)
        out.b2(k, j, i) = base.b2(k, j, i) - (c3 * (B.e1(k + 1, j, i) - B.e1(k, j, i)) -
                                              c1 * (B.e3(k, j, i + 1) - B.e3(k, j, i)));
      else
        out.b2(k, j, i) = base.b2(k, j, i) + c1 * (B.e3(k, j, i + 1) - B.e3(k, j, i));
    });
    const int kb3 = d3 ? g.ke + 1 : 2;
    par3(Bounds{g.ks, kb3, g.js, g.je, g.is, g.ie}, [&](int k, int j, int i) {
      const int ke = d3 ? k : 0;  // 2D: both layers use the k = 0 edge values
      out.b3(k, j, i) = base.b3(k, j, i) - (c1 * (B.e2(ke, j, i + 1) - B.e2(ke, j, i)) -
                                            c2 * (B.e1(ke, j + 1, i) - B.e1(ke, j, i)));
    });
    // end-of-stage cons_to_prim over active cells; floors fix u
    par3(active(), [&](int k, int j, int i) {
      R u[NHYDRO], b[3], w[NCONS];
      for (int v = 0; v < NHYDRO; ++v) u[v] = out.u[v](k, j, i);
      bcc(out, k, j, i, b);
      const int fl = cons_to_prim(u, b, ph, w, true);
      if (fl & 3) {
        nfloor->fetch_add(((fl & 1) ? 1 : 0) + ((fl & 2) ? 1 : 0));
        for (int v = 0; v < NHYDRO; ++v) out.u[v](k, j, i) = u[v];
      }
      if (fl & 4) record_bad(B, k, j, i, bad);
      for (int v = 0; v < NCONS; ++v) B.wend[v](k, j, i) = w[v];
    });
  }

  // compute_dt: min over active cells and dims of
  // dx_d / (|v_d| + c_f,d), times CFL.  min is exact, so any fold order gives
  // the same bits.
  R dt_min_block(const Field<R>* w) const {
    using std::fabs; using std::fmin;
    R m = R(1.0e300);
    for (int k = g.ks; k < g.ke; ++k)
      for (int j = g.js; j < g.je; ++j)
        for (int i = g.is; i < g.ie; ++i) {
          const R d = w[IDN](k, j, i), p = w[IPR](k, j, i);
          const R b1 = w[IB1](k, j, i), b2 = w[IB2](k, j, i), b3 = w[IB3](k, j, i);
          const R c1 = fast_speed_n(d, p, b1, b2, b3, ph.gamma);
          const R c2 = fast_speed_n(d, p, b2, b3, b1, ph.gamma);
          R t = fmin(g.dx[0] / (fabs(w[IV1](k, j, i)) + c1), g.dx[1] / (fabs(w[IV2](k, j, i)) + c2));
          if (g.dim == 3) {
            const R c3 = fast_speed_n(d, p, b3, b1, b2, ph.gamma);
            t = fmin(t, g.dx[2] / (fabs(w[IV3](k, j, i)) + c3));
          }
          m = fmin(m, t);
        }
    return m;
  }

  //--------------------------------------------------------------------------
  // exchange_ghosts: sequential periodic sweeps x1, x2, x3;
  // each sweep writes only ghost layers of its own direction and reads only
  // active layers, so corners and edges fill in order.
  // Normal face-B: lower ghost faces [0, s] take the lower neighbour's
  // [e-ng, e] (the shared face is owned by the lower-index block,
  // SPEC.md:100); upper ghost faces [e+1, e+ng] take the upper neighbour's
  // [s+1, s+ng].
  void exchange(bool use_B) {
    for (int dir = 0; dir < g.dim; ++dir) sweep(dir, use_B);
  }

  //--------------------------------------------------------------------------
  // Turbulence driving (definition in include/pmhd_host.h,
  // GPU: kernels_drive.cu).  dv per local block on active cells; sums per
  // block: each (k, j) row summed over i, each k plane over its rows in j
  // order, the block over its planes in k order.
  std::vector<Field<R>> dvel;  // 3 per local block

  void drive_begin(int nmode, const int* kv, const double* cv, const double* sv,
                   const double* const* ct, const double* const* st, double* sums) {
    dvel.assign(3 * blocks.size(), Field<R>());
    for (size_t b = 0; b < blocks.size(); ++b) {
      Block<R>& B = blocks[b];
      Field<R>* D = &dvel[3 * b];
      for (int a = 0; a < 3; ++a) D[a].resize(g.n[2], g.n[1], g.n[0]);
      R s0 = R(0.0), s1 = R(0.0), s2 = R(0.0), s3 = R(0.0);
      for (int k = g.ks; k < g.ke; ++k) {
        R p0 = R(0.0), p1 = R(0.0), p2 = R(0.0), p3 = R(0.0);  // plane sums (rows in j order)
        for (int j = g.js; j < g.je; ++j) {
          R r0 = R(0.0), r1 = R(0.0), r2 = R(0.0), r3 = R(0.0);
          for (int i = g.is; i < g.ie; ++i) {
            const int gi = B.c[0] * g.mb[0] + (i - g.is), gj = B.c[1] * g.mb[1] + (j - g.js);
            const int gk = (g.dim == 3) ? B.c[2] * g.mb[2] + (k - g.ks) : 0;
            R dv0 = R(0.0), dv1 = R(0.0), dv2 = R(0.0);
            for (int m = 0; m < nmode; ++m) {
              const int qx = (kv[3 * m] + 2) * g.nx[0] + gi;
              const int qy = (kv[3 * m + 1] + 2) * g.nx[1] + gj;
              const int qz = (kv[3 * m + 2] + 2) * g.nx[2] + gk;
              const R axr = ct[0][qx], axi = st[0][qx], ayr = ct[1][qy], ayi = st[1][qy];
              const R azr = ct[2][qz], azi = st[2][qz];
              const R zr = axr * ayr - axi * ayi, zi = axr * ayi + axi * ayr;
              const R cr = zr * azr - zi * azi, ci = zr * azi + zi * azr;
              dv0 = dv0 + (cv[3 * m] * cr + sv[3 * m] * ci);
              dv1 = dv1 + (cv[3 * m + 1] * cr + sv[3 * m + 1] * ci);
              dv2 = dv2 + (cv[3 * m + 2] * cr + sv[3 * m + 2] * ci);
            }
            D[0](k, j, i) = dv0;
            D[1](k, j, i) = dv1;
            D[2](k, j, i) = dv2;
            const R rho = B.A.u[IDN](k, j, i);
            r0 = r0 + rho;
            r1 = r1 + rho * dv0;
            r2 = r2 + rho * dv1;
            r3 = r3 + rho * dv2;
          }
          p0 = p0 + r0; p1 = p1 + r1; p2 = p2 + r2; p3 = p3 + r3;
        }
        s0 = s0 + p0; s1 = s1 + p1; s2 = s2 + p2; s3 = s3 + p3;
      }
      sums[4 * b] = value_of(s0); sums[4 * b + 1] = value_of(s1); sums[4 * b + 2] = value_of(s2); sums[4 * b + 3] = value_of(s3);
    }
  }

  void drive_energy(const double* mean, double* sums) {
    for (size_t b = 0; b < blocks.size(); ++b) {
      Block<R>& B = blocks[b];
      const Field<R>* D = &dvel[3 * b];
      R s0 = R(0.0), s1 = R(0.0);
      for (int k = g.ks; k < g.ke; ++k) {
        R p0 = R(0.0), p1 = R(0.0);
        for (int j = g.js; j < g.je; ++j) {
          R r0 = R(0.0), r1 = R(0.0);
          for (int i = g.is; i < g.ie; ++i) {
            const R rho = B.A.u[IDN](k, j, i);
            const R p0 = D[0](k, j, i) - mean[0], p1 = D[1](k, j, i) - mean[1], p2 = D[2](k, j, i) - mean[2];
            const R q = p0 * p0 + p1 * p1 + p2 * p2;
            r0 = r0 + 0.5 * rho * q;
            r1 = r1 + (B.A.u[IM1](k, j, i) * p0 + B.A.u[IM2](k, j, i) * p1 + B.A.u[IM3](k, j, i) * p2);
          }
          p0 = p0 + r0; p1 = p1 + r1;
        }
        s0 = s0 + p0; s1 = s1 + p1;
      }
      sums[4 * b] = value_of(s0); sums[4 * b + 1] = value_of(s1); sums[4 * b + 2] = 0.0; sums[4 * b + 3] = 0.0;
    }
  }

  void drive_apply(const double* mean, double scale) {
    for (size_t b = 0; b < blocks.size(); ++b) {
      Block<R>& B = blocks[b];
      const Field<R>* D = &dvel[3 * b];
      for (int k = g.ks; k < g.ke; ++k)
        for (int j = g.js; j < g.je; ++j)
          for (int i = g.is; i < g.ie; ++i) {
            const R rho = B.A.u[IDN](k, j, i);
            const R p0 = D[0](k, j, i) - mean[0], p1 = D[1](k, j, i) - mean[1], p2 = D[2](k, j, i) - mean[2];
            const R a0 = B.A.u[IM1](k, j, i), a1 = B.A.u[IM2](k, j, i), a2 = B.A.u[IM3](k, j, i);
            const R sr = scale * rho;
            const R n0 = a0 + sr * p0, n1 = a1 + sr * p1, n2 = a2 + sr * p2;
            const R irho = 1.0 / rho;
            const R ke0 = 0.5 * (a0 * a0 + a1 * a1 + a2 * a2) * irho;
            const R ke1 = 0.5 * (n0 * n0 + n1 * n1 + n2 * n2) * irho;
            B.A.u[IM1](k, j, i) = n0;
            B.A.u[IM2](k, j, i) = n1;
            B.A.u[IM3](k, j, i) = n2;
            B.A.u[IEN](k, j, i) = B.A.u[IEN](k, j, i) + (ke1 - ke0);
          }
    }
    exchange(false);
  }

  // Ghost range that block side r receives in direction dir, for array v
  // (0..4 cells, 5..7 faces b1f..b3f): [q0, q1) along dir.  The sender's
  // range is the same shifted by +m (r = 0, from the lower neighbour) or -m.
  void recv_range(int dir, int r, int v, int* q0, int* q1) const {
    const int ng = g.ng, s = (dir == 0) ? g.is : (dir == 1 ? g.js : g.ks), e = s + g.mb[dir];
    const bool normal = (v == 5 + dir);
    if (r == 0) { *q0 = 0; *q1 = normal ? s + 1 : ng; }
    else { *q0 = normal ? e + 1 : e; *q1 = e + ng + (normal ? 1 : 0); }
  }
  static Field<R>& field(State<R>& S, int v) { return v < 5 ? S.u[v] : (v == 5 ? S.b1 : (v == 6 ? S.b2 : S.b3)); }
  static const Field<R>& field(const State<R>& S, int v) {
    return v < 5 ? S.u[v] : (v == 5 ? S.b1 : (v == 6 ? S.b2 : S.b3));
  }
  int neighbour(const Block<R>& blk, int dir, int side) const {
    int c[3] = {blk.c[0], blk.c[1], blk.c[2]};
    c[dir] += side ? 1 : -1;
    return g.gid_of(c);
  }

  // One sweep over the blocks whose neighbour is local; ghosts facing a
  // remote neighbour are left for unpack().
  void sweep(int dir, bool use_B) {
    const int m = g.mb[dir];
    for (auto& blk : blocks) {
      State<R>& D = use_B ? blk.B : blk.A;
      for (int r = 0; r < 2; ++r) {
        const int ln = local_of[neighbour(blk, dir, r)];
        if (ln < 0) continue;
        const State<R>& N = use_B ? blocks[ln].B : blocks[ln].A;
        for (int v = 0; v < 8; ++v) {
          int q0, q1;
          recv_range(dir, r, v, &q0, &q1);
          copy_slab(field(D, v), field(N, v), dir, q0, q1, r == 0 ? m : -m);
        }
      }
    }
  }

  // pack_boundary: the slab block gid sends to its neighbour
  // on `side` in direction dir; variable-major (u0..u4, b1f, b2f, b3f), each
  // slab in k-j-i order with i fastest.  Returns the element count.
  template <class Fn>
  static void for_slab(const Field<R>& f, int dir, int q0, int q1, Fn&& fn) {
    const int kb = (dir == 2) ? q0 : 0, kend = (dir == 2) ? q1 : f.n3;
    const int jb = (dir == 1) ? q0 : 0, jend = (dir == 1) ? q1 : f.n2;
    const int ib = (dir == 0) ? q0 : 0, iend = (dir == 0) ? q1 : f.n1;
    for (int k = kb; k < kend; ++k)
      for (int j = jb; j < jend; ++j)
        for (int i = ib; i < iend; ++i) fn(k, j, i);
  }
  size_t pack(int gid, int dir, int side, bool use_B, double* out) {
    const Block<R>& blk = blocks[local_of[gid]];
    const State<R>& S = use_B ? blk.B : blk.A;
    const int r = 1 - side, m = g.mb[dir];
    size_t n = 0;
    for (int v = 0; v < 8; ++v) {
      int q0, q1;
      recv_range(dir, r, v, &q0, &q1);
      const int sh = (r == 0) ? m : -m;  // receiver q <- sender q + sh
      const Field<R>& f = field(S, v);
      for_slab(f, dir, q0 + sh, q1 + sh, [&](int k, int j, int i) { out[n++] = value_of(f(k, j, i)); });
    }
    return n;
  }
  // unpack_boundary: ghosts of block gid on `side` (0 lower,
  // 1 upper) from the neighbour's pack(..., 1 - side).
  size_t unpack(int gid, int dir, int side, bool use_B, const double* in) {
    Block<R>& blk = blocks[local_of[gid]];
    State<R>& S = use_B ? blk.B : blk.A;
    size_t n = 0;
    for (int v = 0; v < 8; ++v) {
      int q0, q1;
      recv_range(dir, side, v, &q0, &q1);
      Field<R>& f = field(S, v);
      for_slab(f, dir, q0, q1, [&](int k, int j, int i) { f(k, j, i) = R(in[n++]); });
    }
    return n;
  }
  size_t halo_count(int dir, int side) const {
    size_t n = 0;
    const int ext[8][3] = {{g.n[0], g.n[1], g.n[2]}, {g.n[0], g.n[1], g.n[2]}, {g.n[0], g.n[1], g.n[2]},
                           {g.n[0], g.n[1], g.n[2]}, {g.n[0], g.n[1], g.n[2]},
                           {g.n[0] + 1, g.n[1], g.n[2]}, {g.n[0], g.n[1] + 1, g.n[2]},
                           {g.n[0], g.n[1], g.n[2] + 1}};
    for (int v = 0; v < 8; ++v) {
      int q0, q1;
      recv_range(dir, side, v, &q0, &q1);
      size_t t = 1;
      for (int a = 0; a < 3; ++a) t *= (a == dir) ? size_t(q1 - q0) : size_t(ext[v][a]);
      n += t;
    }
    return n;
  }

  // dst[idx_dir = q] = src[q + off] for q in [q0, q1), all other indices full.
  static void copy_slab(Field<R>& dst, const Field<R>& src, int dir, int q0, int q1, int off) {
    const int kb = (dir == 2) ? q0 : 0, kend = (dir == 2) ? q1 : dst.n3;
    const int jb = (dir == 1) ? q0 : 0, jend = (dir == 1) ? q1 : dst.n2;
    const int ib = (dir == 0) ? q0 : 0, iend = (dir == 0) ? q1 : dst.n1;
    const int ok = (dir == 2) ? off : 0, oj = (dir == 1) ? off : 0, oi = (dir == 0) ? off : 0;
    for (int k = kb; k < kend; ++k)
      for (int j = jb; j < jend; ++j)
        for (int i = ib; i < iend; ++i) dst(k, j, i) = src(k + ok, j + oj, i + oi);
  }

  //--------------------------------------------------------------------------
  // One VL2 stage.  Stage 1: B = A - (dt/2) L_donor(A).
  // Stage 2: A = A - dt L_plm(B).  Then exchange the result.  *bad receives
  // the smallest failing global cell key (unchanged if none).
  void stage(int s, double dt, std::atomic<long long>* bad, std::atomic<long long>* nfloor,
             bool do_exchange = true) {
    for (auto& B : blocks) {
      const State<R>& in = (s == 1) ? B.A : B.B;
      const double f0 = g_tally.total();
      c2p_all(B, in, bad);
      const double f1 = g_tally.total();
      for (int dir = 0; dir < g.dim; ++dir) fluxes(B, in, dir, s == 2, dt);  // splits [1] / [2]
      const double f2 = g_tally.total();
      emfs(B);
      const double f3 = g_tally.total();
      State<R>& out = (s == 1) ? B.B : B.A;
      update(B, B.A, out, (s == 1) ? 0.5 : 1.0, dt, bad, nfloor);
      g_region[0] += f1 - f0;  // (the tally only moves in counting meshes)
      g_region[3] += f3 - f2;
      g_region[4] += g_tally.total() - f3;
    }
    if (do_exchange) exchange(s == 1);
  }

  // dt after stage 2 (from the end-of-stage primitives), CFL * min.
  R new_dt_from_wend() const {
    using std::fmin;
    R m = R(1.0e300);
    for (const auto& B : blocks) m = fmin(m, dt_min_block(B.wend));
    return cfl * m;
  }
  // dt of the state A (initial dt).
  R new_dt_from_state(std::atomic<long long>* bad) {
    using std::fmin;
    R m = R(1.0e300);
    for (auto& B : blocks) {
      c2p_all(B, B.A, bad);
      m = fmin(m, dt_min_block(B.w));
    }
    return cfl * m;
  }
};

}  // namespace oracle

#endif
