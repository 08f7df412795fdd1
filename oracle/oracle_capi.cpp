// oracle/oracle_capi.cpp -- TEST INFRASTRUCTURE, not product code.
//
// C API over the CPU oracle (pmhd_oracle.hpp) so that tests/, smoke() and the
// bench cpu_baseline leg can drive it with the same calls they make on the
// product ABI (include/pmhd_gpu.h).  The op names mirror the reference ops:
// vl2_step / exchange_ghosts / compute_dt / max_divergence_b (SPEC.md:73-90,
// :159-167, :209-217).
#include <atomic>
#include <climits>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pmhd_oracle.hpp"

using oracle::Counting;
using oracle::Mesh;

namespace {

thread_local std::string g_err = "";

struct MeshBase {
  virtual ~MeshBase() = default;
  virtual const oracle::Geometry& geom() const = 0;
  virtual void set_block(int gid, const double* u, const double* b1, const double* b2,
                         const double* b3) = 0;
  virtual void get_block(int gid, double* u, double* w, double* b1, double* b2, double* b3) = 0;
  virtual void exchange() = 0;
  virtual double new_dt(std::atomic<long long>* bad) = 0;
  virtual void stage(int s, double dt, std::atomic<long long>* bad, std::atomic<long long>* nf) = 0;
  virtual long long take_fallbacks() = 0;
  virtual double dt_after_stage2() = 0;
  virtual void diag(int kind, double* out) = 0;
  virtual void face_data(int gid, int dir, double* out) = 0;
  virtual void emf_data(int gid, int comp, double* out) = 0;
  virtual void stage_nx(int s, double dt, std::atomic<long long>* bad, std::atomic<long long>* nf) = 0;
  virtual void sweep(int dir, bool half) = 0;
  virtual size_t halo_count(int dir, int side) const = 0;
  virtual size_t pack(int gid, int dir, int side, bool half, double* out) = 0;
  virtual size_t unpack(int gid, int dir, int side, bool half, const double* in) = 0;
  virtual int local_of(int gid) const = 0;
  virtual void drive_begin(int n, const int* k, const double* c, const double* s, const double* const* ct,
                           const double* const* st, double* sums) = 0;
  virtual void drive_energy(const double* mean, double* sums) = 0;
  virtual void drive_apply(const double* mean, double scale) = 0;
};

template <class R>
struct MeshImpl final : MeshBase {
  Mesh<R> m;
  MeshImpl(const pmhd_mesh_desc& d, std::vector<int> gids) : m(d, std::move(gids)) {}
  void stage_nx(int s, double dt, std::atomic<long long>* bad, std::atomic<long long>* nf) override {
    m.stage(s, dt, bad, nf, false);
  }
  void sweep(int dir, bool half) override { m.sweep(dir, half); }
  void drive_begin(int n, const int* k, const double* c, const double* s, const double* const* ct,
                   const double* const* st, double* sums) override {
    m.drive_begin(n, k, c, s, ct, st, sums);
  }
  void drive_energy(const double* mean, double* sums) override { m.drive_energy(mean, sums); }
  void drive_apply(const double* mean, double scale) override { m.drive_apply(mean, scale); }
  size_t halo_count(int dir, int side) const override { return m.halo_count(dir, side); }
  size_t pack(int gid, int dir, int side, bool half, double* out) override {
    return m.pack(gid, dir, side, half, out);
  }
  size_t unpack(int gid, int dir, int side, bool half, const double* in) override {
    return m.unpack(gid, dir, side, half, in);
  }
  int local_of(int gid) const override { return m.local_of[gid]; }
  const oracle::Geometry& geom() const override { return m.g; }

  static void load(oracle::Field<R>& f, const double* src) {
    for (size_t n = 0; n < f.a.size(); ++n) f.a[n] = R(src[n]);
  }
  static void store(const oracle::Field<R>& f, double* dst) {
    for (size_t n = 0; n < f.a.size(); ++n) dst[n] = oracle::value_of(f.a[n]);
  }

  void set_block(int gid, const double* u, const double* b1, const double* b2,
                 const double* b3) override {
    auto& S = m.blocks[m.local_of[gid]].A;
    const size_t nc = S.u[0].a.size();
    for (int v = 0; v < oracle::NHYDRO; ++v) load(S.u[v], u + v * nc);
    load(S.b1, b1); load(S.b2, b2); load(S.b3, b3);
  }
  void get_block(int gid, double* u, double* w, double* b1, double* b2, double* b3) override {
    auto& B = m.blocks[m.local_of[gid]];
    auto& S = B.A;
    const auto& g = m.g;
    const size_t nc = S.u[0].a.size();
    if (u) {
      for (int v = 0; v < oracle::NHYDRO; ++v) store(S.u[v], u + v * nc);
      for (int k = 0; k < g.n[2]; ++k)
        for (int j = 0; j < g.n[1]; ++j)
          for (int i = 0; i < g.n[0]; ++i) {
            R b[3];
            Mesh<R>::bcc(S, k, j, i, b);
            const size_t idx = (size_t(k) * g.n[1] + j) * g.n[0] + i;
            for (int c = 0; c < 3; ++c) u[(5 + c) * nc + idx] = oracle::value_of(b[c]);
          }
    }
    if (w) {
      std::atomic<long long> bad{LLONG_MAX};
      m.c2p_all(B, S, &bad);
      for (int v = 0; v < oracle::NCONS; ++v) store(B.w[v], w + v * nc);
    }
    if (b1) store(S.b1, b1);
    if (b2) store(S.b2, b2);
    if (b3) store(S.b3, b3);
  }
  void exchange() override { m.exchange(false); }
  double new_dt(std::atomic<long long>* bad) override { return oracle::value_of(m.new_dt_from_state(bad)); }
  long long take_fallbacks() override { return m.fallbacks.exchange(0); }
  void stage(int s, double dt, std::atomic<long long>* bad, std::atomic<long long>* nf) override {
    m.stage(s, dt, bad, nf);
  }
  double dt_after_stage2() override { return oracle::value_of(m.new_dt_from_wend()); }
  void diag(int kind, double* out) override {
    const auto& g = m.g;
    if (kind == PMHD_DIAG_DIVB_MAX) {
      double mx = 0.0;
      for (const auto& B : m.blocks) {
        const auto& S = B.A;
        for (int k = g.ks; k < g.ke; ++k)
          for (int j = g.js; j < g.je; ++j)
            for (int i = g.is; i < g.ie; ++i) {
              double d = (oracle::value_of(S.b1(k, j, i + 1)) - oracle::value_of(S.b1(k, j, i))) / g.dx[0] +
                         (oracle::value_of(S.b2(k, j + 1, i)) - oracle::value_of(S.b2(k, j, i))) / g.dx[1] +
                         (oracle::value_of(S.b3(k + 1, j, i)) - oracle::value_of(S.b3(k, j, i))) / g.dx[2];
              mx = std::fmax(mx, std::fabs(d));
            }
      }
      out[0] = mx;
    } else {
      for (int v = 0; v < 5; ++v) out[v] = 0.0;
      for (const auto& B : m.blocks) {
        // fixed order: row sums over i, then rows in (k, j) order, then blocks
        double s[5] = {0, 0, 0, 0, 0};
        for (int k = g.ks; k < g.ke; ++k)
          for (int j = g.js; j < g.je; ++j)
            for (int v = 0; v < 5; ++v) {
              double r = 0.0;
              for (int i = g.is; i < g.ie; ++i) r += oracle::value_of(B.A.u[v](k, j, i));
              s[v] += r;
            }
        for (int v = 0; v < 5; ++v) out[v] += s[v];
      }
    }
  }
  void face_data(int gid, int dir, double* out) override {
    const auto& B = m.blocks[m.local_of[gid]];
    const size_t nf = B.fx[dir][0].a.size();
    for (int v = 0; v < 8; ++v) store(B.fx[dir][v], out + v * nf);
  }
  void emf_data(int gid, int comp, double* out) override {
    const auto& B = m.blocks[m.local_of[gid]];
    store(comp == 0 ? B.e1 : (comp == 1 ? B.e2 : B.e3), out);
  }
};

void fill_status(const oracle::Geometry& g, long long bad, int stage, long long nf, pmhd_status* st,
                 long long fb = 0) {
  if (!st) return;
  st->floor_count = nf;
  st->fallback_count = fb;
  st->stage = stage;
  if (bad == LLONG_MAX) {
    st->code = PMHD_OK; st->k = st->j = st->i = -1;
  } else {
    st->code = PMHD_ERR_UNPHYSICAL;
    st->i = int(bad % g.nx[0]);
    st->j = int((bad / g.nx[0]) % g.nx[1]);
    st->k = int(bad / (long long)(g.nx[0]) / g.nx[1]);
  }
}

}  // namespace

struct oracle_mesh {
  std::unique_ptr<MeshBase> impl;
  bool counting = false;
};

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

// gids / n_local: the blocks this (rank's) mesh owns; n_local <= 0: all.
int oracle_mesh_create_local(const pmhd_mesh_desc* d, int counting, int workers, const int* gids,
                             int n_local, oracle_mesh** out) {
  try {
    std::vector<int> g;
    for (int b = 0; b < n_local; ++b) g.push_back(gids[b]);
    auto* m = new oracle_mesh;
    if (counting) m->impl.reset(new MeshImpl<Counting>(*d, g));
    else m->impl.reset(new MeshImpl<double>(*d, g));
    m->counting = counting != 0;
    oracle::g_workers = counting ? 1 : (workers < 1 ? 1 : workers);
    *out = m;
    return PMHD_OK;
  } catch (const oracle::ConfigErr& e) {
    g_err = e.what();
    return PMHD_ERR_CONFIG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PMHD_ERR_INPUT;
  }
}

int oracle_mesh_create(const pmhd_mesh_desc* d, int counting, int workers, oracle_mesh** out) {
  return oracle_mesh_create_local(d, counting, workers, nullptr, 0, out);
}

void oracle_mesh_destroy(oracle_mesh* m) { delete m; }

int oracle_is_local(oracle_mesh* m, int gid) {
  return (gid >= 0 && gid < m->impl->geom().nblocks && m->impl->local_of(gid) >= 0) ? 1 : 0;
}

// Multi-rank pieces: a stage without its trailing exchange, one local sweep,
// and pack/unpack of the halo slabs facing remote neighbours.
// half = 1 selects the u^{n+1/2} state (after stage 1), 0 the u^n state.
int oracle_stage_compute(oracle_mesh* m, int stage, double dt, double* dt_next, pmhd_status* st) {
  if (stage != 1 && stage != 2) { g_err = "stage must be 1 or 2"; return PMHD_ERR_INPUT; }
  std::atomic<long long> bad{LLONG_MAX}, nf{0};
  m->impl->stage_nx(stage, dt, &bad, &nf);
  if (stage == 2 && dt_next) *dt_next = m->impl->dt_after_stage2();
  fill_status(m->impl->geom(), bad.load(), stage, nf.load(), st, m->impl->take_fallbacks());
  return bad.load() == LLONG_MAX ? PMHD_OK : PMHD_ERR_UNPHYSICAL;
}
int oracle_exchange_dir(oracle_mesh* m, int dir, int half) { m->impl->sweep(dir, half != 0); return PMHD_OK; }
long long oracle_halo_count(oracle_mesh* m, int dir, int side) { return (long long)m->impl->halo_count(dir, side); }
int oracle_halo_pack(oracle_mesh* m, int gid, int dir, int side, int half, double* out) {
  if (!oracle_is_local(m, gid)) { g_err = "block not local"; return PMHD_ERR_INPUT; }
  m->impl->pack(gid, dir, side, half != 0, out);
  return PMHD_OK;
}
int oracle_halo_unpack(oracle_mesh* m, int gid, int dir, int side, int half, const double* in) {
  if (!oracle_is_local(m, gid)) { g_err = "block not local"; return PMHD_ERR_INPUT; }
  m->impl->unpack(gid, dir, side, half != 0, in);
  return PMHD_OK;
}

void oracle_set_workers(int workers) { oracle::g_workers = workers < 1 ? 1 : workers; }

int oracle_block_dims(oracle_mesh* m, int n[3]) {
  const auto& g = m->impl->geom();
  n[0] = g.n[0]; n[1] = g.n[1]; n[2] = g.n[2];
  return PMHD_OK;
}

int oracle_nblocks(oracle_mesh* m) { return m->impl->geom().nblocks; }
int oracle_nlocal(oracle_mesh* m) {
  int n = 0;
  for (int g = 0; g < m->impl->geom().nblocks; ++g) n += (m->impl->local_of(g) >= 0);
  return n;
}

int oracle_set_block(oracle_mesh* m, int gid, const double* u, const double* b1, const double* b2,
                     const double* b3) {
  if (!oracle_is_local(m, gid)) { g_err = "bad gid"; return PMHD_ERR_INPUT; }
  m->impl->set_block(gid, u, b1, b2, b3);
  return PMHD_OK;
}

int oracle_get_block(oracle_mesh* m, int gid, double* u, double* w, double* b1, double* b2,
                     double* b3) {
  if (!oracle_is_local(m, gid)) { g_err = "bad gid"; return PMHD_ERR_INPUT; }
  m->impl->get_block(gid, u, w, b1, b2, b3);
  return PMHD_OK;
}

int oracle_exchange(oracle_mesh* m) { m->impl->exchange(); return PMHD_OK; }

int oracle_new_dt(oracle_mesh* m, double* dt, pmhd_status* st) {
  std::atomic<long long> bad{LLONG_MAX};
  *dt = m->impl->new_dt(&bad);
  fill_status(m->impl->geom(), bad.load(), 0, 0, st);
  return bad.load() == LLONG_MAX ? PMHD_OK : PMHD_ERR_UNPHYSICAL;
}

int oracle_stage(oracle_mesh* m, int stage, double dt, double* dt_next, pmhd_status* st) {
  if (stage != 1 && stage != 2) { g_err = "stage must be 1 or 2"; return PMHD_ERR_INPUT; }
  std::atomic<long long> bad{LLONG_MAX}, nf{0};
  m->impl->stage(stage, dt, &bad, &nf);
  if (stage == 2 && dt_next) *dt_next = m->impl->dt_after_stage2();
  fill_status(m->impl->geom(), bad.load(), stage, nf.load(), st, m->impl->take_fallbacks());
  return bad.load() == LLONG_MAX ? PMHD_OK : PMHD_ERR_UNPHYSICAL;
}

int oracle_vl2_step(oracle_mesh* m, double dt, double* dt_next, pmhd_status* st) {
  pmhd_status s1;
  int rc = oracle_stage(m, 1, dt, nullptr, &s1);
  if (rc != PMHD_OK) { if (st) *st = s1; return rc; }
  rc = oracle_stage(m, 2, dt, dt_next, st);
  if (st) { st->floor_count += s1.floor_count; st->fallback_count += s1.fallback_count; }
  return rc;
}

int oracle_diag(oracle_mesh* m, int kind, double* out) {
  if (kind != PMHD_DIAG_DIVB_MAX && kind != PMHD_DIAG_SUMS) { g_err = "bad diag"; return PMHD_ERR_INPUT; }
  m->impl->diag(kind, out);
  return PMHD_OK;
}

// Face data of the LAST stage of a block: 8 arrays (5 lab-order hydro fluxes,
// ey, ez, weight) with the face-array extents of direction dir.
int oracle_face_data(oracle_mesh* m, int gid, int dir, double* out) {
  m->impl->face_data(gid, dir, out);
  return PMHD_OK;
}
int oracle_emf_data(oracle_mesh* m, int gid, int comp, double* out) {
  m->impl->emf_data(gid, comp, out);
  return PMHD_OK;
}

// Turbulence driving (pmhd_gpu.h drive_* semantics, CPU restatement).
int oracle_drive_begin(oracle_mesh* m, int n, const int* k, const double* c, const double* s,
                       const double* const* ct, const double* const* st, double* sums) {
  m->impl->drive_begin(n, k, c, s, ct, st, sums);
  return PMHD_OK;
}
int oracle_drive_energy(oracle_mesh* m, const double* mean, double* sums) {
  m->impl->drive_energy(mean, sums);
  return PMHD_OK;
}
int oracle_drive_apply(oracle_mesh* m, const double* mean, double scale) {
  m->impl->drive_apply(mean, scale);
  return PMHD_OK;
}

// Flop tally of counting meshes (counting.hpp:31-41 FlopCounts).
void oracle_flops(double out[4]) {
  out[0] = oracle::g_tally.add; out[1] = oracle::g_tally.mul;
  out[2] = oracle::g_tally.div; out[3] = oracle::g_tally.sqrt_n;
}
void oracle_flops_reset(void) {
  oracle::g_tally.reset();
  for (double& r : oracle::g_region) r = 0.0;
}
// out[0..4] = c2p, reconstruct, riemann, ct_emf, integrate (counting.hpp).
void oracle_region_flops(double out[5]) {
  for (int q = 0; q < 5; ++q) out[q] = oracle::g_region[q];
}

//---------------------------------------------------------------- pointwise ops
static pmhd_mesh_desc desc_for(double gamma, int riemann, int limiter) {
  pmhd_mesh_desc d;
  std::memset(&d, 0, sizeof(d));
  d.gamma = gamma; d.riemann = riemann; d.limiter = limiter;
  d.eos_mode = PMHD_EOS_ERROR; d.emf_mode = PMHD_EMF_UPWIND;
  return d;
}

// cons_to_prim of an 8-variable conserved state; returns 0
// or PMHD_ERR_UNPHYSICAL.
int oracle_cons_to_prim(const double* u8, double gamma, double* w8) {
  const oracle::Phys ph(desc_for(gamma, 0, 0));
  double u[5];
  for (int v = 0; v < 5; ++v) u[v] = u8[v];
  const int fl = oracle::cons_to_prim(u, u8 + 5, ph, w8, false);
  return (fl & 4) ? PMHD_ERR_UNPHYSICAL : PMHD_OK;
}

void oracle_prim_to_cons(const double* w8, double gamma, double* u8) {
  const oracle::Phys ph(desc_for(gamma, 0, 0));
  oracle::prim_to_cons(w8, ph, u8);
}

// fast_speed along dim (0,1,2) of an 8-variable primitive state.
double oracle_fast_speed(const double* w8, double gamma, int dim) {
  const int n = 5 + dim, t1 = 5 + (dim + 1) % 3, t2 = 5 + (dim + 2) % 3;
  return oracle::fast_speed_n(w8[0], w8[4], w8[n], w8[t1], w8[t2], gamma);
}

// Riemann flux of rotated states (d, vn, vt1, vt2, p, bt1, bt2); out[0..6] =
// flux of (d, mn, mt1, mt2, e, bt1, bt2).
int oracle_riemann(int solver, const double* wl, const double* wr, double bx, double gamma,
                   double* out) {
  const oracle::Phys ph(desc_for(gamma, solver, 0));
  if (solver == PMHD_RIEMANN_HLLE) oracle::riemann_hlle(wl, wr, bx, ph, out);
  else if (solver == PMHD_RIEMANN_ROE) {
    if (!oracle::riemann_roe(wl, wr, bx, ph, out)) { oracle::riemann_hlle(wl, wr, bx, ph, out); return 1; }
  } else oracle::riemann_hlld(wl, wr, bx, ph, out);
  return 0;
}

double oracle_plm_slope(double qm, double q0, double qp, int limiter) {
  return oracle::plm_slope(qm, q0, qp, limiter);
}

}  // extern "C"

extern "C" {
// Physical 1-D flux F(W) of a rotated state (the side_state flux).
void oracle_phys_flux(const double* w7, double bx, double gamma, double* out7) {
  const oracle::Phys ph(desc_for(gamma, 0, 0));
  oracle::SideState<double> s;
  oracle::side_state(w7, bx, bx * bx, ph, s);
  for (int n = 0; n < 7; ++n) out7[n] = s.f[n];
}
}
