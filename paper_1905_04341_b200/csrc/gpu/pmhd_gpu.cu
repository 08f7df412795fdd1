// pmhd_gpu.cu -- implementation of the C ABI (include/pmhd_gpu.h).
//
// Owns all device memory through opaque handles; host pointers are borrowed
// for the duration of a call.  Each call returns once its results are visible
// to the next call (the par_for synchronization-point contract,
// /root/reference/proj/include/pmhd/exec/dispatch.hpp:106-108).  No C++
// exception crosses the ABI; errors map to the defs.hpp:36-76 families.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include <cudaTypedefs.h>

#include "pmhd_gpu.h"

using namespace pmhd_gpu;

#ifndef PMHD_VARIANT
// (no commas: the string is the policy column of the CLI's CSV row)
#define PMHD_VARIANT "fused(flux: tile + march; update: edge EMF + cell) [PMHD_KERNELS=split: one kernel per op]"
#endif
#ifdef PMHD_BOUNDS_CHECK
#define PMHD_CHECK_INFO "+bounds-check"
#else
#define PMHD_CHECK_INFO ""
#endif
#if defined(PMHD_DIVSQRT_1ULP) && !defined(PMHD_PARITY)
#define PMHD_DS_INFO "+divsqrt(1ulp)"
#else
#define PMHD_DS_INFO ""
#endif
#ifdef PMHD_PARITY
#define PMHD_BUILD_INFO PMHD_VARIANT "+parity(fmad=false)" PMHD_CHECK_INFO
#else
#define PMHD_BUILD_INFO PMHD_VARIANT "+fma" PMHD_DS_INFO PMHD_CHECK_INFO
#endif

struct pmhd_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // update kernels of the k-slab pipeline
  cudaStream_t stream3 = nullptr;  // concurrent flux launches (PMHD_FLUX_CONC=3)
  std::string err;
};

struct pmhd_mesh {
  pmhd_ctx* ctx = nullptr;
  pmhd_mesh_desc desc;
  KGeom G;
  KPhys ph;
  std::vector<int> gids;          // global id of each local block
  std::vector<DevBlock> hblk, hblk_alt;   // current table and its st[0]<->st[2] swap
  DevBlock* dblk = nullptr;
  DevBlock* dblk_alt = nullptr;
  double* slab = nullptr;
  size_t arr_elems = 0;
  size_t per_block = 0;            // doubles per block in the slab
  DevRed* dred = nullptr;         // 3 slots
  DevRed* hred = nullptr;         // pinned mirror
  double* drows = nullptr;
  bool all_local = true;
  bool prof = false;
  bool async_ops = false;         // pmhd_gpu_set_async: stream-ordered multi-rank calls
  // interior-tile prefetch (overlap of a stage's flux work with the previous
  // stage's ghost exchange): stage whose interior flux tiles are enqueued on
  // stream2, with the dt they used; ev_pre[0] = input ready, [1] = done
  // device copies of the stage coefficients (dks[1], dks[2]) and the run
  // control of a graph-replayed pmhd_gpu_run; graphs cached per table parity
  CUtensorMap* ec_maps = nullptr;  // TMA maps of the cell-E arrays (3 per block; nullptr: plain loads)
  // TMA-staged update kernel (3D, PMHD_UPDATE=tma): per table parity, per
  // block, the maps of kernels_update_tma.cu; nullptr = the LDG update kernel
  CUtensorMap* upd_maps = nullptr;
  unsigned long long upd_xoff = 0;
  KStage* dks = nullptr;
  DevCtl* dctl = nullptr;
  int parity = 0;                 // table flips mod 2 (hblk/dblk vs their alternates)
  cudaGraphExec_t gexec[2] = {};  // two cycles each, starting from parity 0 / 1
  int graphs = 2;                 // graph-replayed run: 2 auto (small meshes), PMHD_GRAPH=0/1
  int prefetched = 0;
  double prefetch_dt = 0.0;
  cudaEvent_t ev_pre[2] = {};
  bool overlap = false;           // on for meshes with remote neighbours; PMHD_OVERLAP=0/1 overrides
  // turbulence driving buffers (allocated at the first event)
  double* drive_tab = nullptr;    // 3 axes x (cos, sin) x 5 x nx[a]
  double* drive_rows = nullptr;   // nb x rows x 4, then nb x planes x 4
  double* drive_sums = nullptr;   // nb x 4
  DriveTabs drive{};
  int variant = 0;                // 0: fused flux kernels; 1: split (debug; PMHD_KERNELS=split)
  int slab_planes = 0;            // k-slab pipeline depth (PMHD_SLAB_PLANES, 0 = off)
  bool push_x1 = false;           // update kernel writes the x1 ghosts (PMHD_PUSH_X1, default on when possible)
  bool face_reuse = false;        // flux tiles cover owned faces only + rim images (PMHD_FACE_REUSE)
  FluxOpts fopt;                  // flux kernel choices (PMHD_FACE_REUSE / _FLUX_MARCH / _FLUX_MARCH_X1 / _FLUX_SMEM_PAD)
  int flux_xy = 0;                // x1 + x2 in one launch, bit s-1 for stage s (PMHD_FLUX_XY=1|2|3)
  // flux launches of a stage on two streams (3D, whole-mesh launches): x2 on
  // stream2 beside x1 -> x3 on the main stream fills each launch's tail wave
  // (+0.6-0.8 % at 256^3). PMHD_FLUX_CONC: 0 off, 1 x2 (default), 2 x3, 3 x2 and x3
  int flux_conc = 1;
  cudaEvent_t ev_fx[3] = {};
  // stage-1 x2 / x3 ghost exchanges on stream3, overlapping the stage-2 x1
  // flux launch (which reads no x2 / x3 ghosts with owned-face reuse); the
  // x2 / x3 flux launches wait for ev_ex[d].  PMHD_EARLY_X1: 0 off, 1 on
  // meshes up to 2^24 cells per rank (default), 2 always.
  int early_x1 = 1;
  bool ex_pending = false;
  cudaEvent_t ev_ex[3] = {};
  // stage update: 2 two kernels (edge EMFs + cell update; default, see
  // update_emf_fills), 0 fused (PMHD_UPDATE=ldg), 1
  // warp-specialised (=ws), 3 two kernels always (=emf); tma: upd_maps
  int upd_kind = 2;
  bool emf_rim = true;            // edge EMFs: upper-rim edges stored by the neighbours (PMHD_EMF_RIM=0: formed locally)
  std::vector<cudaEvent_t> slab_ev;
  cudaEvent_t ev[8] = {};
  cudaEvent_t xev[25] = {};        // host<->device transfer pipeline (one per staged array + 1)
  pmhd_region_times times{};
};

namespace {

#define CK(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);          \
      return PMHD_ERR_CUDA;                                                    \
    }                                                                          \
  } while (0)
// CK inside pmhd_gpu_mesh_create once the mesh exists: free what was
// allocated so far (every handle starts null) before returning
#define MCK(call)                                                              \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);          \
      pmhd_gpu_mesh_destroy(m);                                                \
      return PMHD_ERR_CUDA;                                                    \
    }                                                                          \
  } while (0)

int fail(pmhd_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

std::string validate(const pmhd_mesh_desc& d) {
  if (d.ng < 2 || d.ng > 4) return "ng must be in [2, 4]";
  for (int a = 0; a < 3; ++a) {
    if (d.nx[a] < 1 || d.mb[a] < 1) return "cell counts must be positive";
    if (d.nx[a] % d.mb[a] != 0) return "global cells not divisible by meshblock cells";
    if (!(d.xmax[a] > d.xmin[a])) return "empty domain extent";
  }
  if (d.nx[1] == 1) return "1D meshes are not supported";
  if (d.mb[0] <= d.ng || d.mb[1] <= d.ng || (d.nx[2] > 1 && d.mb[2] <= d.ng))
    return "meshblock must have more than ng cells per dimension";
  if (!(d.gamma > 1.0)) return "gamma must be > 1";
  if (!(d.cfl > 0.0 && d.cfl < 1.0)) return "cfl must be in (0,1)";
  if (d.riemann != PMHD_RIEMANN_HLLD && d.riemann != PMHD_RIEMANN_HLLE && d.riemann != PMHD_RIEMANN_ROE)
    return "bad riemann";
  if (d.limiter != PMHD_LIMITER_MC && d.limiter != PMHD_LIMITER_VANLEER) return "bad limiter";
  if (d.eos_mode != PMHD_EOS_ERROR && d.eos_mode != PMHD_EOS_FLOOR) return "bad eos_mode";
  if (d.emf_mode != PMHD_EMF_UPWIND && d.emf_mode != PMHD_EMF_ARITH) return "bad emf_mode";
  return "";
}

void decode_key(const KGeom& G, unsigned long long key, pmhd_status* st) {
  st->i = int(key % (unsigned long long)G.nx[0]);
  st->j = int((key / (unsigned long long)G.nx[0]) % (unsigned long long)G.nx[1]);
  st->k = int(key / (unsigned long long)G.nx[0] / (unsigned long long)G.nx[1]);
}

double bits2d(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof(d));
  return d;
}

int reset_red(pmhd_mesh* m) {
  pmhd_ctx* ctx = m->ctx;
  for (int s = 0; s < 3; ++s) {
    m->hred[s].dt_bits = 0x7FF0000000000000ULL;  // +inf
    m->hred[s].bad_key = ULLONG_MAX;
    m->hred[s].floor_count = 0;
    m->hred[s].divb_bits = 0;
    m->hred[s].fallback_count = 0;
    for (int q = 0; q < 5; ++q) m->hred[s].phase[q] = 0;
  }
  CK(cudaMemcpyAsync(m->dred, m->hred, 3 * sizeof(DevRed), cudaMemcpyHostToDevice, ctx->stream));
  return PMHD_OK;
}

int fetch_red(pmhd_mesh* m) {
  pmhd_ctx* ctx = m->ctx;
  CK(cudaMemcpyAsync(m->hred, m->dred, 3 * sizeof(DevRed), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  return PMHD_OK;
}

void rec(pmhd_mesh* m, int slot) {
  if (m->prof) cudaEventRecord(m->ev[slot], m->ctx->stream);
}

// TMA tensor maps of every block's 3 cell-E arrays for the update kernel's E
// ring: 3D (i, j, k) over the pitched array, box = the kernel's E box.  The
// map starts at element i = -1 so that its base is 16-byte aligned (rows are
// aligned at i = is-1 = 1, i.e. i = -1 is on a 16 B boundary).
int build_ec_maps(pmhd_mesh* m) {
  if (!update_uses_tma()) return PMHD_OK;
  if (const char* t = std::getenv("PMHD_TMA")) if (std::atoi(t) == 0) return PMHD_OK;
  pmhd_ctx* ctx = m->ctx;
  const KGeom& G = m->G;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return PMHD_OK;  // no driver entry point: the kernel uses plain loads
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  int box[2];
  update_ec_box(box);
  std::vector<CUtensorMap> maps(3 * size_t(G.nb));
  for (int b = 0; b < G.nb; ++b)
    for (int c = 0; c < 3; ++c) {
      double* base = m->hblk[b].ec[c] - 1;
      if (reinterpret_cast<uintptr_t>(base) % 16) return PMHD_OK;
      const cuuint64_t dim[3] = {cuuint64_t(G.n1 + 1), cuuint64_t(G.n2), cuuint64_t(G.n3)};
      const cuuint64_t stride[2] = {cuuint64_t(G.sx) * 8, cuuint64_t(G.sy) * 8};
      const cuuint32_t bx[3] = {cuuint32_t(box[0]), cuuint32_t(box[1]), 1};
      const cuuint32_t es[3] = {1, 1, 1};
      const CUresult r = encode(&maps[3 * b + c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dim, stride, bx, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(ctx, PMHD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    }
  CK(cudaMalloc(&m->ec_maps, maps.size() * sizeof(CUtensorMap)));
  CK(cudaMemcpy(m->ec_maps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  return PMHD_OK;
}

// Tensor maps of the TMA-staged update kernel, for both block tables (the
// tables swap u^n and u^{n+1} every cycle): 3D over each pitched array,
// dims (n1+1 [+1], n2+1, n3+1), one box shape per map id.  A map whose
// array is not 16 B aligned starts one element early (bit set in upd_xoff).
// Box starts must be 16 B aligned too: if the row alignment does not give
// that (PMHD_ROW_SHIFT* overrides), no maps are built and the LDG update
// kernel runs.
int build_update_maps(pmhd_mesh* m) {
  const KGeom& G = m->G;
  if (G.dim != 3) return PMHD_OK;
  // opt-in (PMHD_UPDATE=tma): measured slower than the LDG kernel at 256^3
  // (1.64 vs 1.55 ms per launch)
  const char* u = std::getenv("PMHD_UPDATE");
  if (!u || std::string(u) != "tma") return PMHD_OK;
  pmhd_ctx* ctx = m->ctx;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return PMHD_OK;  // no driver entry point: the LDG update kernel
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int per = update_tma_maps_per_block();
  std::vector<CUtensorMap> maps(size_t(2) * G.nb * per);
  unsigned long long xoff = 0;
  for (int par = 0; par < 2; ++par)
    for (int b = 0; b < G.nb; ++b)
      for (int a = 0; a < per; ++a) {
        const DevBlock& B = (par == 0 ? m->hblk : m->hblk_alt)[b];
        const double* arr = update_tma_array(B, a);
        const int xo = int((reinterpret_cast<uintptr_t>(arr) / 8) & 1);
        if (par == 0 && b == 0) xoff |= (unsigned long long)xo << a;
        else if (((xoff >> a) & 1ull) != (unsigned long long)xo) return PMHD_OK;  // (never: uniform shifts)
        int box[3];
        update_tma_box(a, box);
        // every box starts on a 16 B boundary: tile origins are is + 32 n, so
        // the element parity of (is + first cell) must put it there
        if (((reinterpret_cast<uintptr_t>(arr) / 8) + unsigned(G.is + box[2])) & 1u) return PMHD_OK;
        const cuuint64_t dim[3] = {cuuint64_t(G.n1 + 1 + xo), cuuint64_t(G.n2 + 1), cuuint64_t(G.n3 + 1)};
        const cuuint64_t stride[2] = {cuuint64_t(G.sx) * 8, cuuint64_t(G.sy) * 8};
        const cuuint32_t bx[3] = {cuuint32_t(box[0]), cuuint32_t(box[1]), 1};
        const cuuint32_t es[3] = {1, 1, 1};
        const CUresult r = encode(&maps[(size_t(par) * G.nb + b) * per + a], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                                  const_cast<double*>(arr - xo), dim, stride, bx, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(ctx, PMHD_ERR_CUDA, "cuTensorMapEncodeTiled (update maps) failed");
      }
  CK(cudaMalloc(&m->upd_maps, maps.size() * sizeof(CUtensorMap)));
  CK(cudaMemcpy(m->upd_maps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  m->upd_xoff = xoff;
  return PMHD_OK;
}

// Whether the stage update runs as the two kernels (edge EMFs + cell update)
bool update_two_kernels(const pmhd_mesh* m, int kr0, int kr1) {
  return !m->upd_maps && m->G.dim >= 2 && m->ph.prof == 0 &&
         (m->upd_kind == 3 || (m->upd_kind == 2 && update_emf_fills(m->G, kr0, kr1)));
}

// The update of one stage over planes [kr0, kr1): the TMA-staged kernel when
// its maps exist (3D, PMHD_UPDATE=tma), the two kernels (default), the
// warp-specialised kernel (PMHD_UPDATE=ws) or the fused LDG kernel.
void launch_update_any(pmhd_mesh* m, const KStage& ks, const KStage* kd, int want_dt, int kr0, int kr1,
                       cudaStream_t st, int push) {
  if (m->upd_maps) {
    const CUtensorMap* maps = m->upd_maps + size_t(m->parity) * m->G.nb * update_tma_maps_per_block();
    launch_update_tma(m->dblk, m->G, m->ph, ks, kd, m->dred, want_dt, kr0, kr1, st, maps, m->upd_xoff, push);
  } else if (update_two_kernels(m, kr0, kr1)) {
    // two kernels: corner EMFs, then the cell update (not under phase
    // profiling, which splits the fused kernel's time by its phases)
    launch_update_emf(m->dblk, m->G, m->ph, ks, kd, m->dred, want_dt, kr0, kr1, st, push,
                      (m->all_local && m->emf_rim) ? 1 : 0);
  } else if (m->G.dim == 3 && m->upd_kind == 1) {
    launch_update_ws(m->dblk, m->G, m->ph, ks, kd, m->dred, want_dt, kr0, kr1, st, push);
  } else {
    launch_update_fused(m->dblk, m->G, m->ph, ks, kd, m->dred, want_dt, kr0, kr1, st, m->ec_maps, push);
  }
}

KStage make_stage(const KGeom& G, int s, double dt) {
  const double beta = (s == 1) ? 0.5 : 1.0;
  const double bdt = beta * dt;
  KStage ks;
  ks.c1 = bdt / G.dx[0];
  ks.c2 = bdt / G.dx[1];
  ks.c3 = bdt / G.dx[2];
  for (int d = 0; d < 3; ++d) ks.c1024[d] = 1024.0 * dt / G.dx[d];
  ks.in_sel = (s == 1) ? 0 : 1;
  ks.out_sel = (s == 1) ? 1 : 2;
  ks.stage = s;
  ks.plm = (s == 2);
  ks.skip = 0;
  return ks;
}

bool can_prefetch(const pmhd_mesh* m) { return m->overlap && m->variant == 0 && !m->prof; }

// x1 and x2 faces in one k_flux_xy launch (PMHD_FLUX_XY=1): owned-face
// ranges only (the two directions then share one tile grid)
bool use_flux_xy(const pmhd_mesh* m, int s) {
  // opt-in: measured 6.6 % slower at 256^3 in both stages (16 warps/SM);
  // PMHD_FLUX_XY=1: both stages, 2: stage 1 only (bit 0), 3: both
  return m->variant == 0 && m->face_reuse && ((m->flux_xy >> (s - 1)) & 1);
}

// Interior flux tiles of stage s on stream2, after the work already on the
// main stream (the update that produced their input); the ghost exchange that
// follows on the main stream runs concurrently (the tiles read no ghost data).
int prefetch_stage(pmhd_mesh* m, int s, double dt) {
  pmhd_ctx* ctx = m->ctx;
  const KGeom& G = m->G;
  const KStage ks = make_stage(G, s, dt);
  CK(cudaEventRecord(m->ev_pre[0], ctx->stream));
  CK(cudaStreamWaitEvent(ctx->stream2, m->ev_pre[0], 0));
  for (int dir = 0; dir < G.dim; ++dir)
    launch_flux_fused(m->dblk, G, m->ph, dir, ks.in_sel, ks.plm, ks.c1024[dir], nullptr, s, m->dred, 0,
                      1, G.ke - G.ks, ctx->stream2, 1, m->fopt);
  CK(cudaEventRecord(m->ev_pre[1], ctx->stream2));
  m->times.kernel_launches += G.dim;
  m->prefetched = s;
  m->prefetch_dt = dt;
  CK(cudaGetLastError());
  return PMHD_OK;
}

// Enqueue one VL2 stage (no synchronization unless profiling).
// prefetch_next: enqueue the next stage's interior flux tiles (same dt) on
// stream2 before this stage's exchange, so they overlap it.
// device_ks: the kernels read the coefficients (and the skip flag) from the
// device copy k_cycle_begin writes in a captured cycle; else by value.
int enqueue_stage(pmhd_mesh* m, int s, double dt, bool do_exchange = true, bool prefetch_next = false,
                  bool device_ks = false, bool early_ok = false) {
  pmhd_ctx* ctx = m->ctx;
  const KGeom& G = m->G;
  const KStage ks = make_stage(G, s, dt);
  const KStage* kd = device_ks ? m->dks + s : nullptr;
  cudaStream_t st = ctx->stream;
  // interior tiles of this stage already enqueued (with this dt)?
  int flux_region = 0;
  if (m->prefetched) {
    if (m->prefetched == s && m->prefetch_dt == dt && can_prefetch(m)) flux_region = 2;
    CK(cudaStreamWaitEvent(st, m->ev_pre[1], 0));  // (a stale prefetch must finish before it is redone)
    m->prefetched = 0;
  }
  // k-slab pipeline (fused variant, 3D, not profiling): the flux kernels of
  // slab q+1 run on the main stream while the update kernel of slab q (which
  // needs the faces of planes up to the first plane of slab q+1) runs on the
  // second stream, overlapping the FP64-bound flux work with the
  // memory-bound update work.
  const int nk = G.ke - G.ks;
  int S = nk, nslab = 1;
  if (m->variant == 0 && G.dim == 3 && !m->prof && m->slab_planes > 0 && nk >= 2 * m->slab_planes &&
      flux_region == 0) {
    S = m->slab_planes;
    nslab = (nk + S - 1) / S;
  }
  if (nslab > 1) {
    for (int q = 0; q < nslab; ++q) {
      for (int dir = 0; dir < G.dim; ++dir)
        launch_flux_fused(m->dblk, G, m->ph, dir, ks.in_sel, ks.plm, ks.c1024[dir], kd, s, m->dred, q,
                          nslab, S, st);
      CK(cudaEventRecord(m->slab_ev[q], st));
      if (q >= 1) {  // update slab q-1 once the flux kernels of slab q are done
        CK(cudaStreamWaitEvent(ctx->stream2, m->slab_ev[q], 0));
        launch_update_any(m, ks, kd, s == 2, G.ks + (q - 1) * S, G.ks + q * S, ctx->stream2, 0);
      }
    }
    CK(cudaStreamWaitEvent(ctx->stream2, m->slab_ev[nslab - 1], 0));
    launch_update_any(m, ks, kd, s == 2, G.ks + (nslab - 1) * S, G.ke, ctx->stream2, 0);
    CK(cudaEventRecord(m->slab_ev[nslab], ctx->stream2));
    CK(cudaStreamWaitEvent(st, m->slab_ev[nslab], 0));
    if (do_exchange) launch_exchange(m->dblk, G, ks.out_sel, st, kd);
    m->times.kernel_launches += nslab * ((update_two_kernels(m, G.ks, G.ks + S) ? 2 : 1) + G.dim) +
                                (do_exchange ? G.dim : 0);
  } else {
    rec(m, 0);
    if (m->variant == 1) launch_c2p_all(m->dblk, G, m->ph, ks.in_sel, m->dred, s, st);
    rec(m, 1);
    const bool xy = use_flux_xy(m, s) && flux_region == 0;
    if (xy) launch_flux_xy(m->dblk, G, m->ph, ks.in_sel, ks.plm, ks.c1024[0], ks.c1024[1], kd, s, m->dred, st);
    // concurrent flux launches (PMHD_FLUX_CONC, opt-in): one direction on
    // stream2 beside the other two on the main stream, joined before the update
    const int cdir = (m->flux_conc && m->variant == 0 && flux_region == 0 && !xy && !m->prof &&
                      (G.dim == 3 || (G.dim == 2 && m->flux_conc == 1)))
                         ? m->flux_conc : -1;
    // stream of each direction's flux launch
    cudaStream_t fst[3] = {st, st, st};
    if (cdir == 1 || cdir == 3) fst[1] = ctx->stream2;
    if (cdir == 2) fst[2] = ctx->stream2;
    if (cdir == 3) fst[2] = ctx->stream3;
    if (cdir > 0) {
      CK(cudaEventRecord(m->ev_fx[0], st));
      CK(cudaStreamWaitEvent(ctx->stream2, m->ev_fx[0], 0));
      if (cdir == 3) CK(cudaStreamWaitEvent(ctx->stream3, m->ev_fx[0], 0));
    }
    for (int dir = xy ? 2 : 0; dir < G.dim; ++dir) {
      // a pending stage-1 exchange of direction dir must be done first (x1:
      // pushed by the update kernel, no wait)
      if (m->ex_pending && dir >= 1) CK(cudaStreamWaitEvent(fst[dir], m->ev_ex[dir], 0));
      if (m->variant == 0)
        launch_flux_fused(m->dblk, G, m->ph, dir, ks.in_sel, ks.plm, ks.c1024[dir], kd, s, m->dred, 0, 1,
                          nk, fst[dir], flux_region, m->fopt);
      else
        launch_flux(m->dblk, G, m->ph, dir, ks.in_sel, ks.plm, ks.c1024[dir], st);
    }
    if (m->ex_pending) {  // (joined through the x2 / x3 launches; stream3 fully)
      CK(cudaStreamWaitEvent(st, m->ev_ex[G.dim - 1], 0));
      m->ex_pending = false;
    }
    if (cdir > 0) {
      CK(cudaEventRecord(m->ev_fx[1], ctx->stream2));
      CK(cudaStreamWaitEvent(st, m->ev_fx[1], 0));
      if (cdir == 3) {
        CK(cudaEventRecord(m->ev_fx[2], ctx->stream3));
        CK(cudaStreamWaitEvent(st, m->ev_fx[2], 0));
      }
    }
    rec(m, 2);
    if (m->variant == 1) launch_emf(m->dblk, G, m->ph, st);
    rec(m, 3);
    if (m->variant == 0) {
      launch_update_any(m, ks, kd, s == 2, G.ks, G.ke, st, m->push_x1 ? 1 : 0);
    } else {
      launch_update(m->dblk, G, ks, st);
      launch_c2p_end(m->dblk, G, m->ph, ks, m->dred, s == 2, st);
    }
    rec(m, 4);
    if (do_exchange && prefetch_next && s == 1 && can_prefetch(m)) {
      int rc = prefetch_stage(m, 2, dt);
      if (rc) return rc;
    }
    // (x1 ghosts already stored by the update kernel when pushed)
    const int d0 = (m->variant == 0 && m->push_x1) ? 1 : 0;
    // stage 1 of a step: the x2 / x3 exchanges on stream3, so the stage-2 x1
    // flux launch (owned faces only: no x2 / x3 ghosts read) overlaps them
    // (not with the fused x1 + x2 launch of stage 2, which needs the x2
    // ghosts; measured +2 % on the 64^3 wave, +1 % on 512^2 Orszag-Tang, 0 to
    // +0.2 % at 256^3 and -0.2 % on the 512^3 turbulence in 64 blocks, so
    // meshes up to 2^24 cells per rank; PMHD_EARLY_X1=0 / 2: never / always)
    const long long cells = (long long)G.mb[0] * G.mb[1] * G.mb[2] * G.nb;
    // stage 2: the exchanges overlap the next step's stage-1 x1 flux launch
    // (every other entry point that touches the state joins them first:
    // drop_prefetch, run, destroy)
    const bool early = early_ok && do_exchange && d0 == 1 && m->face_reuse && m->variant == 0 && !m->prof &&
                       !can_prefetch(m) && !use_flux_xy(m, s == 1 ? 2 : 1) &&
                       (m->early_x1 == 2 || (m->early_x1 == 1 && cells <= (1LL << 24)));
    if (early) {
      CK(cudaEventRecord(m->ev_ex[0], st));
      CK(cudaStreamWaitEvent(ctx->stream3, m->ev_ex[0], 0));
      for (int dir = 1; dir < G.dim; ++dir) {
        launch_exchange_dir(m->dblk, G, ks.out_sel, dir, ctx->stream3, kd);
        CK(cudaEventRecord(m->ev_ex[dir], ctx->stream3));
      }
      m->ex_pending = true;
    } else if (do_exchange) {
      for (int dir = d0; dir < G.dim; ++dir) launch_exchange_dir(m->dblk, G, ks.out_sel, dir, st, kd);
    }
    rec(m, 5);
    const int nupd = update_two_kernels(m, G.ks, G.ke) ? 2 : 1;
    m->times.kernel_launches += ((m->variant == 0) ? nupd + G.dim - (xy ? 1 : 0) : 4 + G.dim) + (do_exchange ? G.dim - d0 : 0);
  }
  CK(cudaGetLastError());
  if (s == 2) {  // u^{n+1} (st[2]) becomes the current state: flip the tables
    std::swap(m->hblk, m->hblk_alt);
    std::swap(m->dblk, m->dblk_alt);
    m->parity ^= 1;
  }
  if (m->prof) {
    CK(cudaEventSynchronize(m->ev[5]));
    float t[5];
    for (int q = 0; q < 5; ++q) cudaEventElapsedTime(&t[q], m->ev[q], m->ev[q + 1]);
    double c2p = t[0], rec_ms = 0.0, rie = t[1], emf = t[2], integ = t[3];
    if (m->variant == 0) {
      // fused kernels: split each kernel's event time by the SM-cycle shares
      // of its phases (clock64 at the kernels' barriers, summed over CTAs)
      int rc = fetch_red(m);
      if (rc) return rc;
      const unsigned long long* ph = m->hred[s].phase;
      const double pf = double(ph[0]) + double(ph[1]) + double(ph[2]);
      const double pu = double(ph[3]) + double(ph[4]);
      if (pf > 0.0) {
        c2p += t[1] * double(ph[0]) / pf;
        rec_ms = t[1] * double(ph[1]) / pf;
        rie = t[1] * double(ph[2]) / pf;
      }
      if (pu > 0.0) {
        emf += t[3] * double(ph[3]) / pu;
        integ = t[3] * double(ph[4]) / pu;
      }
    }
    m->times.c2p_ms += c2p;
    m->times.reconstruct_ms += rec_ms;
    m->times.riemann_ms += rie;
    m->times.ct_emf_ms += emf;
    m->times.integrate_ms += integ;
    m->times.boundary_ms += t[4];
    m->times.calls += 1;
  }
  return PMHD_OK;
}

int finish(pmhd_mesh* m, int stage_lo, int stage_hi, double* dt_next, pmhd_status* st) {
  int rc = fetch_red(m);
  if (rc) return rc;
  pmhd_status s{};
  s.code = PMHD_OK;
  s.k = s.j = s.i = -1;
  s.stage = stage_hi;
  long long nf = 0;
  long long fb = 0;
  for (int q = stage_lo; q <= stage_hi; ++q) nf += (long long)m->hred[q].floor_count;
  for (int q = stage_lo; q <= stage_hi; ++q) fb += (long long)m->hred[q].fallback_count;
  s.floor_count = nf;
  s.fallback_count = fb;
  for (int q = stage_lo; q <= stage_hi; ++q) {
    if (m->hred[q].bad_key != ULLONG_MAX) {
      s.code = PMHD_ERR_UNPHYSICAL;
      s.stage = q;
      decode_key(m->G, m->hred[q].bad_key, &s);
      break;
    }
  }
  if (dt_next) *dt_next = m->desc.cfl * bits2d(m->hred[0].dt_bits);
  if (st) *st = s;
  if (s.code != PMHD_OK) {
    m->ctx->err = "unphysical state in stage " + std::to_string(s.stage);
    return PMHD_ERR_UNPHYSICAL;
  }
  return PMHD_OK;
}

// A pending stage prefetch (interior flux tiles on stream2) writes the
// face-data arrays the transfers stage through and accumulates into the
// reduction slots: the main stream waits for it, and its fluxes are void
// afterwards (the next stage recomputes every tile).
int drop_prefetch(pmhd_mesh* m) {
  pmhd_ctx* ctx = m->ctx;
  if (m->prefetched) {
    CK(cudaStreamWaitEvent(ctx->stream, m->ev_pre[1], 0));
    m->prefetched = 0;
  }
  if (m->ex_pending) {  // ghost exchanges still running beside the main stream
    CK(cudaStreamWaitEvent(ctx->stream, m->ev_ex[m->G.dim - 1], 0));
    m->ex_pending = false;
  }
  return PMHD_OK;
}

int local_index(const pmhd_mesh* m, int gid) {
  for (size_t b = 0; b < m->gids.size(); ++b)
    if (m->gids[b] == gid) return int(b);
  return -1;
}

// Empty kernel: cudaFuncGetAttributes on it fails unless this library's
// sm_100a image loads on the device (pmhd_gpu_ctx_create).
__global__ void k_image_probe() {}

// Every ABI call that touches the device makes the context's device current
// first: the caller may have switched devices between calls.
int use_device(pmhd_ctx* ctx) {
  CK(cudaSetDevice(ctx->device));
  return PMHD_OK;
}

}  // namespace

extern "C" {

int pmhd_gpu_abi_version(void) { return PMHD_ABI_VERSION; }

const char* pmhd_gpu_build_info(void) { return PMHD_BUILD_INFO; }

int pmhd_gpu_ctx_create(int device, pmhd_ctx** out) {
  if (!out) return PMHD_ERR_INPUT;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) return PMHD_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return PMHD_ERR_CUDA;
  // built for sm_100a only: arch-specific code loads on compute capability
  // 10.0 alone, so a 10.x part other than 10.0 is refused here rather than
  // at the first launch ("no kernel image"); the probe confirms the image
  // loads on this device
  if (prop.major != 10 || prop.minor != 0) return PMHD_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return PMHD_ERR_CUDA;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_image_probe) != cudaSuccess) {
    cudaGetLastError();
    return PMHD_ERR_CUDA;
  }
  auto* ctx = new pmhd_ctx;
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->stream3, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return PMHD_ERR_CUDA;
  }
  *out = ctx;
  return PMHD_OK;
}

int pmhd_gpu_ctx_destroy(pmhd_ctx* ctx) {
  if (!ctx) return PMHD_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  if (ctx->stream3) cudaStreamDestroy(ctx->stream3);
  delete ctx;
  return PMHD_OK;
}

const char* pmhd_gpu_last_error(const pmhd_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

int pmhd_gpu_mesh_create(pmhd_ctx* ctx, const pmhd_mesh_desc* desc, const int* gids, int n_local,
                         pmhd_mesh** out) {
  if (!ctx || !desc || !out) return PMHD_ERR_INPUT;
  *out = nullptr;
  const std::string v = validate(*desc);
  if (!v.empty()) return fail(ctx, PMHD_ERR_CONFIG, v);
  CK(cudaSetDevice(ctx->device));
  auto* m = new pmhd_mesh;
  m->ctx = ctx;
  m->desc = *desc;
  KGeom& G = m->G;
  G.dim = (desc->nx[2] == 1) ? 2 : 3;
  G.ng = desc->ng;
  int nb[3];
  for (int a = 0; a < 3; ++a) {
    G.nx[a] = desc->nx[a];
    G.mb[a] = desc->mb[a];
    nb[a] = desc->nx[a] / desc->mb[a];
    G.dx[a] = (desc->xmax[a] - desc->xmin[a]) / desc->nx[a];
  }
  G.n1 = G.mb[0] + 2 * G.ng;
  G.n2 = G.mb[1] + 2 * G.ng;
  G.n3 = (G.dim == 3) ? G.mb[2] + 2 * G.ng : 1;
  {
    // kernels index a block array with 32-bit ints (idx(k,j,i) = k*sy + j*sx + i)
    const long long sx = ((G.n1 + 1 + 31) / 32) * 32, sy = sx * (G.n2 + 1);
    if ((long long)(G.n3 + 1) * sy + 64 >= (1LL << 31)) {
      delete m;
      return fail(ctx, PMHD_ERR_CONFIG, "MeshBlock too large (a block array must hold < 2^31 doubles): use smaller blocks");
    }
    G.sx = int(sx);
    G.sy = int(sy);
  }
  {
    // every kernel serves all local blocks in one launch with the block index
    // folded into gridDim.z together with at most n+1 planes or rows of a
    // block (flux: face planes / rows, update: k segments, split kernels and
    // exchange: planes or 8 arrays); gridDim.z is limited to 65535
    const long long nbl = (n_local <= 0 || !gids)
                              ? (long long)(desc->nx[0] / desc->mb[0]) * (desc->nx[1] / desc->mb[1]) *
                                    (desc->nx[2] / desc->mb[2])
                              : n_local;
    const long long per = std::max({(long long)G.n2, (long long)G.n3, (long long)kNState}) + 1;
    if (nbl * per > 65535) {
      delete m;
      return fail(ctx, PMHD_ERR_CONFIG,
                  "too many MeshBlocks on this rank for their size: (local blocks) x (block cells incl. ghosts "
                  "along x2/x3 + 1) must be <= 65535 (" + std::to_string(nbl) + " x " + std::to_string(per) +
                      "); use larger MeshBlocks or more ranks");
    }
  }
  G.is = G.ng; G.ie = G.ng + G.mb[0];
  G.js = G.ng; G.je = G.ng + G.mb[1];
  if (G.dim == 3) { G.ks = G.ng; G.ke = G.ng + G.mb[2]; } else { G.ks = 0; G.ke = 1; }
  const int ntot = nb[0] * nb[1] * nb[2];
  if (n_local <= 0 || !gids) {
    for (int g = 0; g < ntot; ++g) m->gids.push_back(g);
  } else {
    std::vector<char> seen(ntot, 0);
    for (int b = 0; b < n_local; ++b) {
      if (gids[b] < 0 || gids[b] >= ntot) { delete m; return fail(ctx, PMHD_ERR_CONFIG, "gid out of range"); }
      if (seen[gids[b]]++) { delete m; return fail(ctx, PMHD_ERR_CONFIG, "duplicate gid"); }
      m->gids.push_back(gids[b]);
    }
  }
  G.nb = int(m->gids.size());
  if (const char* kv = std::getenv("PMHD_KERNELS")) m->variant = (std::string(kv) == "split") ? 1 : 0;
  if (const char* sp = std::getenv("PMHD_SLAB_PLANES")) m->slab_planes = std::atoi(sp);
  if (m->slab_planes > 0) m->slab_planes = std::max(16, (m->slab_planes / 16) * 16);  // x3 tile multiple
  m->ph.gamma = desc->gamma;
  m->ph.gm1 = desc->gamma - 1.0;
  m->ph.igm1 = 1.0 / (desc->gamma - 1.0);
  m->ph.dfloor = desc->dfloor;
  m->ph.pfloor = desc->pfloor;
  m->ph.riemann = desc->riemann;
  m->ph.limiter = desc->limiter;
  m->ph.eos = desc->eos_mode;
  m->ph.emf = desc->emf_mode;
  m->ph.prof = 0;

  // one slab: 59 arrays per block, each (n3+1)*sy doubles plus a 64-double guard
  const size_t arr = size_t(G.n3 + 1) * size_t(G.sy) + 64;
  m->arr_elems = arr;
  const size_t per_block = 59 * arr;
  m->per_block = per_block;
  const size_t bytes = per_block * G.nb * sizeof(double);
  if (cudaMalloc(&m->slab, bytes) != cudaSuccess) {
    delete m;
    return fail(ctx, PMHD_ERR_CUDA, "device allocation of " + std::to_string(bytes) + " bytes failed");
  }
  cudaMemsetAsync(m->slab, 0, bytes, ctx->stream);
  m->hblk.resize(G.nb);
  // Row alignment per array group: element i = shift of every row starts a
  // 256 B segment.  State and cell-E rows are aligned at i = is-1 (the first
  // cell the x2/x3 flux tiles and the update's E box touch), face-data rows at
  // i = is (the update tiles' first face); measured best of the (0..2)^3
  // combinations on B200 (+4.7 % over unshifted).  PMHD_ROW_SHIFT[_ST|_FX|_EC]
  // override for experiments.
  auto shift_env = [](const char* k, int d) {
    const char* v = std::getenv(k);
    return v ? std::max(0, std::min(31, std::atoi(v))) : d;
  };
  const int a1 = std::min(31, G.ng - 1), a2 = std::min(31, G.ng);  // i = is-1, i = is
  const int sh_st = shift_env("PMHD_ROW_SHIFT_ST", shift_env("PMHD_ROW_SHIFT", a1));
  const int sh_fx = shift_env("PMHD_ROW_SHIFT_FX", shift_env("PMHD_ROW_SHIFT", a2));
  const int sh_ec = shift_env("PMHD_ROW_SHIFT_EC", shift_env("PMHD_ROW_SHIFT", a1));
  for (int b = 0; b < G.nb; ++b) {
    double* p = m->slab + size_t(b) * per_block + 32;
    m->hblk[b].base = reinterpret_cast<const char*>(m->slab + size_t(b) * per_block);
    DevBlock& B = m->hblk[b];
    auto take = [&](int sh) { double* q = p - sh; p += arr; return q; };
    for (int s = 0; s < 3; ++s)
      for (int v = 0; v < kNState; ++v) B.st[s][v] = take(sh_st);
    for (int v = 0; v < 8; ++v) B.w[v] = take(sh_st);
    for (int d = 0; d < 3; ++d)
      for (int v = 0; v < 8; ++v) B.fx[d][v] = take(sh_fx);
    for (int c = 0; c < 3; ++c) B.e[c] = take(sh_ec);
    for (int c = 0; c < 3; ++c) B.ec[c] = B.e[c];
    const int gid = m->gids[b];
    B.c[0] = gid % nb[0];
    B.c[1] = (gid / nb[0]) % nb[1];
    B.c[2] = gid / (nb[0] * nb[1]);
    for (int d = 0; d < 3; ++d)
      for (int side = 0; side < 2; ++side) {
        int c[3] = {B.c[0], B.c[1], B.c[2]};
        c[d] = (c[d] + (side ? 1 : -1) + nb[d]) % nb[d];
        const int ng = (c[2] * nb[1] + c[1]) * nb[0] + c[0];
        int li = -1;
        for (int q = 0; q < G.nb; ++q) if (m->gids[q] == ng) { li = q; break; }
        if (li < 0) m->all_local = false;  // remote: ghosts come from halo unpack
        B.nbr[d][side] = li;
      }
  }
  // second table with st[0] <-> st[2] swapped (flipped after every cycle)
  m->hblk_alt = m->hblk;
  for (auto& B : m->hblk_alt)
    for (int v = 0; v < kNState; ++v) std::swap(B.st[0][v], B.st[2][v]);
  MCK(cudaMalloc(&m->dblk, sizeof(DevBlock) * G.nb));
  MCK(cudaMalloc(&m->dblk_alt, sizeof(DevBlock) * G.nb));
  MCK(cudaMemcpyAsync(m->dblk, m->hblk.data(), sizeof(DevBlock) * G.nb, cudaMemcpyHostToDevice, ctx->stream));
  MCK(cudaMemcpyAsync(m->dblk_alt, m->hblk_alt.data(), sizeof(DevBlock) * G.nb, cudaMemcpyHostToDevice,
                     ctx->stream));
  MCK(cudaMalloc(&m->dred, 3 * sizeof(DevRed)));
  MCK(cudaMalloc(&m->dks, 3 * sizeof(KStage)));
  if (G.dim == 3) {
    int rc = build_ec_maps(m);
    if (!rc) rc = build_update_maps(m);
    if (rc) { pmhd_gpu_mesh_destroy(m); return rc; }
  }
  MCK(cudaMalloc(&m->dctl, sizeof(DevCtl)));
  MCK(cudaMemsetAsync(m->dks, 0, 3 * sizeof(KStage), ctx->stream));
  if (const char* gr = std::getenv("PMHD_GRAPH")) m->graphs = std::atoi(gr) != 0 ? 1 : 0;
  MCK(cudaMallocHost(&m->hred, 3 * sizeof(DevRed)));
  const size_t nrows = size_t(G.nb) * 5 * (G.ke - G.ks) * (G.je - G.js);
  MCK(cudaMalloc(&m->drows, nrows * sizeof(double)));
  for (auto& e : m->ev) MCK(cudaEventCreate(&e));
  for (auto& e : m->ev_pre) MCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : m->ev_fx) MCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : m->ev_ex) MCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : m->xev) MCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // Overlap pays where the exchange is a real transfer (remote neighbours,
  // NCCL); with all neighbours local the exchange kernels take ~3 % of a
  // stage and splitting the flux launches costs more (measured -1.4 % at 256^3).
  m->overlap = !m->all_local;
  if (const char* ov = std::getenv("PMHD_OVERLAP")) m->overlap = std::atoi(ov) != 0;
  // x1 ghost push: every block's x1 neighbours local and mutual (regular
  // periodic decomposition), so the update kernel can store the x1 ghost
  // layers itself and the in-stage x1 exchange launch is dropped
  m->push_x1 = true;
  for (int b = 0; b < G.nb; ++b) {
    const int L = m->hblk[b].nbr[0][0], R = m->hblk[b].nbr[0][1];
    if (L < 0 || R < 0 || m->hblk[L].nbr[0][1] != b || m->hblk[R].nbr[0][0] != b) m->push_x1 = false;
  }
  if (G.mb[0] < G.ng) m->push_x1 = false;
  if (const char* px = std::getenv("PMHD_PUSH_X1")) m->push_x1 = m->push_x1 && std::atoi(px) != 0;
  // owned-face reuse (kernels_flux.cu): every neighbour local, so every
  // halo face the update reads has an owner on this rank; not with the
  // k-slab pipeline (images cross slabs)
  m->face_reuse = m->all_local && m->slab_planes == 0;
  if (const char* fr = std::getenv("PMHD_FACE_REUSE")) m->face_reuse = m->face_reuse && std::atoi(fr) != 0;
  // the other kernel choices, read once here
  m->fopt.reuse = m->face_reuse ? 1 : 0;
  if (const char* e = std::getenv("PMHD_FLUX_MARCH")) m->fopt.march = std::max(0, std::min(2, std::atoi(e)));
  if (const char* e = std::getenv("PMHD_FLUX_MARCH_X1")) m->fopt.march_x1 = std::atoi(e) != 0 ? 1 : 0;
  if (const char* e = std::getenv("PMHD_FLUX_MARCH_STAGES")) m->fopt.march_stages = std::atoi(e) & 3;
  if (const char* e = std::getenv("PMHD_FLUX_SMEM_PAD")) m->fopt.pad = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("PMHD_FLUX_XY")) m->flux_xy = (std::atoi(e) == 1) ? 3 : (std::atoi(e) & 3);
  if (const char* e = std::getenv("PMHD_EARLY_X1")) m->early_x1 = std::max(0, std::min(2, std::atoi(e)));
  if (const char* e = std::getenv("PMHD_FLUX_CONC")) m->flux_conc = std::max(0, std::min(3, std::atoi(e)));
  if (const char* e = std::getenv("PMHD_EMF_RIM")) m->emf_rim = std::atoi(e) != 0;
  if (const char* e = std::getenv("PMHD_UPDATE"))
    m->upd_kind = (std::string(e) == "ws") ? 1 : (std::string(e) == "emf") ? 3 : 0;
  m->slab_ev.resize((G.ke - G.ks) / 8 + 2);
  for (auto& e : m->slab_ev) MCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  MCK(cudaStreamSynchronize(ctx->stream));
  *out = m;
  return PMHD_OK;
}

int pmhd_gpu_mesh_destroy(pmhd_mesh* m) {
  if (!m) return PMHD_OK;
  cudaSetDevice(m->ctx->device);
  cudaStreamSynchronize(m->ctx->stream);
  cudaStreamSynchronize(m->ctx->stream3);  // (deferred ghost exchanges)
  cudaFree(m->slab);
  if (m->drive_tab) { cudaFree(m->drive_tab); cudaFree(m->drive_rows); cudaFree(m->drive_sums); }
  cudaFree(m->dblk);
  cudaFree(m->dblk_alt);
  cudaFree(m->dred);
  cudaFree(m->dks);
  if (m->ec_maps) cudaFree(m->ec_maps);
  if (m->upd_maps) cudaFree(m->upd_maps);
  cudaFree(m->dctl);
  for (auto& g : m->gexec) if (g) cudaGraphExecDestroy(g);
  cudaFree(m->drows);
  cudaFreeHost(m->hred);
  for (auto& e : m->ev) if (e) cudaEventDestroy(e);
  for (auto& e : m->slab_ev) if (e) cudaEventDestroy(e);
  for (auto& e : m->ev_pre) if (e) cudaEventDestroy(e);
  for (auto& e : m->ev_fx) if (e) cudaEventDestroy(e);
  for (auto& e : m->ev_ex) if (e) cudaEventDestroy(e);
  for (auto& e : m->xev) if (e) cudaEventDestroy(e);
  delete m;
  return PMHD_OK;
}

int pmhd_gpu_block_dims(const pmhd_mesh* m, int n[3]) {
  if (!m || !n) return PMHD_ERR_INPUT;
  n[0] = m->G.n1; n[1] = m->G.n2; n[2] = m->G.n3;
  return PMHD_OK;
}

// One array between a dense host buffer (e1 x e2 x e3, i fastest) and a
// pitched block array, staged through a contiguous device buffer: one large
// PCIe DMA (full speed from pinned memory) plus an HBM-speed repack kernel.
// Host <-> device transfer of a block's arrays through dense staging buffers:
// one PCIe DMA per array at full speed from pinned memory plus an HBM-speed
// repack kernel (pitched <-> dense).  Each array gets its own staging buffer
// (the block's 24 face-data arrays are free outside a stage), so the copies
// run back to back on the copy stream (stream2) while the repack / Bcc
// kernels run on the main stream, ordered per array by events.
struct Xfer {
  double* host;
  const double* dev;  // pitched source / destination (kind 0), face array (kind 1: Bcc)
  int e1, e2, e3;
  int kind, comp;     // kind 1: face_to_center_b of component comp (download only)
};

static int xfer_pipelined(pmhd_mesh* m, DevBlock& B, const Xfer* it, int n, bool to_host) {
  pmhd_ctx* ctx = m->ctx;
  const KGeom& G = m->G;
  if (n > 24) return fail(ctx, PMHD_ERR_INPUT, "too many staged arrays");
  cudaStream_t s = ctx->stream, c = ctx->stream2;
  // the staging buffers may still be in use by work already on the main stream
  CK(cudaEventRecord(m->xev[24], s));
  CK(cudaStreamWaitEvent(c, m->xev[24], 0));
  for (int q = 0; q < n; ++q) {
    double* stg = B.fx[q / 8][q % 8];
    const size_t bytes = size_t(it[q].e1) * it[q].e2 * it[q].e3 * sizeof(double);
    if (to_host) {
      if (it[q].kind == 1) launch_bcc_dense(stg, it[q].dev, G, it[q].comp, s);
      else launch_repack(stg, const_cast<double*>(it[q].dev), G, it[q].e1, it[q].e2, it[q].e3, 1, s);
      CK(cudaGetLastError());
      CK(cudaEventRecord(m->xev[q], s));
      CK(cudaStreamWaitEvent(c, m->xev[q], 0));
      CK(cudaMemcpyAsync(it[q].host, stg, bytes, cudaMemcpyDeviceToHost, c));
    } else {
      CK(cudaMemcpyAsync(stg, it[q].host, bytes, cudaMemcpyHostToDevice, c));
      CK(cudaEventRecord(m->xev[q], c));
      CK(cudaStreamWaitEvent(s, m->xev[q], 0));
      launch_repack(stg, const_cast<double*>(it[q].dev), G, it[q].e1, it[q].e2, it[q].e3, 0, s);
      CK(cudaGetLastError());
    }
  }
  CK(cudaStreamSynchronize(c));
  CK(cudaStreamSynchronize(s));
  return PMHD_OK;
}

int pmhd_gpu_upload_block(pmhd_mesh* m, int gid, const double* u, const double* b1f,
                          const double* b2f, const double* b3f) {
  if (!m) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  pmhd_ctx* ctx = m->ctx;
  const int b = local_index(m, gid);
  if (b < 0) return fail(ctx, PMHD_ERR_INPUT, "block not local");
  if (!u || !b1f || !b2f || !b3f) return fail(ctx, PMHD_ERR_BUFFER, "null buffer");
  if (int rc = drop_prefetch(m)) return rc;
  const KGeom& G = m->G;
  const size_t nc = size_t(G.n1) * G.n2 * G.n3;
  DevBlock& B = m->hblk[b];
  double* hu = const_cast<double*>(u);
  Xfer it[8];
  for (int v = 0; v < 5; ++v) it[v] = {hu + v * nc, B.st[0][v], G.n1, G.n2, G.n3, 0, 0};
  it[5] = {const_cast<double*>(b1f), B.st[0][5], G.n1 + 1, G.n2, G.n3, 0, 0};
  it[6] = {const_cast<double*>(b2f), B.st[0][6], G.n1, G.n2 + 1, G.n3, 0, 0};
  it[7] = {const_cast<double*>(b3f), B.st[0][7], G.n1, G.n2, G.n3 + 1, 0, 0};
  return xfer_pipelined(m, B, it, 8, false);
}

int pmhd_gpu_download_block(pmhd_mesh* m, int gid, double* u, double* w, double* b1f, double* b2f,
                            double* b3f) {
  if (!m) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  pmhd_ctx* ctx = m->ctx;
  const int b = local_index(m, gid);
  if (b < 0) return fail(ctx, PMHD_ERR_INPUT, "block not local");
  if (int rc = drop_prefetch(m)) return rc;
  const KGeom& G = m->G;
  const size_t nc = size_t(G.n1) * G.n2 * G.n3;
  DevBlock& B = m->hblk[b];
  Xfer it[24];
  int n = 0;
  if (u) {
    for (int v = 0; v < 5; ++v) it[n++] = {u + v * nc, B.st[0][v], G.n1, G.n2, G.n3, 0, 0};
    // face_to_center_b on the device, same IEEE operations
    for (int c = 0; c < 3; ++c) it[n++] = {u + (5 + c) * nc, B.st[0][5 + c], G.n1, G.n2, G.n3, 1, c};
  }
  if (b1f) it[n++] = {b1f, B.st[0][5], G.n1 + 1, G.n2, G.n3, 0, 0};
  if (b2f) it[n++] = {b2f, B.st[0][6], G.n1, G.n2 + 1, G.n3, 0, 0};
  if (b3f) it[n++] = {b3f, B.st[0][7], G.n1, G.n2, G.n3 + 1, 0, 0};
  if (w) {
    int rc = reset_red(m);
    if (rc) return rc;
    launch_c2p_all(m->dblk, G, m->ph, 0, m->dred, 0, ctx->stream);
    CK(cudaGetLastError());
    for (int v = 0; v < 8; ++v) it[n++] = {w + v * nc, B.w[v], G.n1, G.n2, G.n3, 0, 0};
  }
  return xfer_pipelined(m, B, it, n, true);
}

int pmhd_gpu_exchange(pmhd_mesh* m) {
  if (!m) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  pmhd_ctx* ctx = m->ctx;
  if (!m->all_local) return fail(ctx, PMHD_ERR_INPUT, "exchange needs all neighbours local");
  if (int rc = drop_prefetch(m)) return rc;
  launch_exchange(m->dblk, m->G, 0, ctx->stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return PMHD_OK;
}

int pmhd_gpu_new_dt(pmhd_mesh* m, double* dt_out, pmhd_status* st) {
  if (!m || !dt_out) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  int rc = drop_prefetch(m);
  if (!rc) rc = reset_red(m);
  if (rc) return rc;
  launch_dt_from_state(m->dblk, m->G, m->ph, m->dred, m->ctx->stream);
  return finish(m, 0, 0, dt_out, st);
}

int pmhd_gpu_stage(pmhd_mesh* m, int stage, double dt, double* dt_next, pmhd_status* st) {
  if (!m) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  if (stage != 1 && stage != 2) return fail(m->ctx, PMHD_ERR_INPUT, "stage must be 1 or 2");
  if (!m->all_local) return fail(m->ctx, PMHD_ERR_INPUT, "stage needs all neighbours local");
  int rc = reset_red(m);
  if (!rc) rc = enqueue_stage(m, stage, dt);
  if (rc) return rc;
  return finish(m, stage, stage, stage == 2 ? dt_next : nullptr, st);
}

int pmhd_gpu_vl2_step(pmhd_mesh* m, double dt, double* dt_next, pmhd_status* st) {
  if (!m) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  if (!m->all_local) return fail(m->ctx, PMHD_ERR_INPUT, "step needs all neighbours local");
  int rc = reset_red(m);
  if (!rc) rc = enqueue_stage(m, 1, dt, true, true, false, true);  // + stage-2 interior tiles over the exchange
  if (!rc) rc = enqueue_stage(m, 2, dt, true, false, false, true);
  if (rc) return rc;
  return finish(m, 1, 2, dt_next, st);
}

namespace {

// The run loop with the cycle on the device: two cycles (one per table parity)
// captured once into a CUDA graph and replayed, with k_cycle_begin/_end
// carrying dt, t, the tlim cap, floors and the first error on the device; the
// host synchronises every 32 cycles instead of every cycle.  Same arithmetic
// as the host loop below, so the same bits.
bool graph_run_ok(const pmhd_mesh* m) {
  if (!(m->graphs != 0 && m->variant == 0 && !m->prof && !m->async_ops && m->all_local &&
        m->slab_planes == 0 && !m->overlap && !m->prefetched))
    return false;
  if (m->graphs == 1) return true;  // PMHD_GRAPH=1
  // auto: where the per-cycle host round trip is a visible share of a cycle
  // (measured: 512^2 and 64^3 +13-15 %; 256^3 -1 %, the device-resident
  // coefficients cost a little latency per CTA)
  const long long cells = (long long)m->G.mb[0] * m->G.mb[1] * m->G.mb[2] * m->G.nb;
  return cells < (1LL << 22);
}

int capture_cycles(pmhd_mesh* m) {
  pmhd_ctx* ctx = m->ctx;
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  int rc = PMHD_OK;
  for (int c = 0; c < 2 && !rc; ++c) {  // two cycles: the tables flip once per cycle
    launch_cycle_begin(m->dctl, m->dks, m->dred, ctx->stream);
    rc = enqueue_stage(m, 1, 0.0, true, false, true, true);
    if (!rc) rc = enqueue_stage(m, 2, 0.0, true, false, true);
    launch_cycle_end(m->dctl, m->dks, m->dred, ctx->stream);
  }
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(ctx, PMHD_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&m->gexec[m->parity], g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(ctx, PMHD_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  return PMHD_OK;
}

int graph_run(pmhd_mesh* m, int ncycles, double tlim, double* t, double* dt, int* cycles_done,
              pmhd_status* st) {
  pmhd_ctx* ctx = m->ctx;
  const KGeom& G = m->G;
  DevCtl c;
  std::memset(&c, 0, sizeof(c));
  c.t = *t;
  c.dt = *dt;
  c.tlim = tlim;
  c.cfl = m->desc.cfl;
  for (int a = 0; a < 3; ++a) c.dx[a] = G.dx[a];
  c.ncycles = ncycles;
  c.stop = ((ncycles >= 0 && ncycles <= 0) || (tlim > 0.0 && *t >= tlim)) ? 1 : 0;
  c.err_key = ULLONG_MAX;
  const int parity0 = m->parity;
  if (!c.stop) {
    if (!m->gexec[parity0]) {
      int rc = capture_cycles(m);  // (capture leaves the tables as they were: two flips)
      if (rc) return rc;
    }
    CK(cudaMemcpyAsync(m->dctl, &c, sizeof(c), cudaMemcpyHostToDevice, ctx->stream));
    while (true) {
      // graph replays (2 cycles each) before the next host check: as many as
      // the cycles left need (a replay past the end costs its skipped
      // launches), at most 16
      int pairs = 16;
      if (ncycles >= 0) pairs = std::min(pairs, (ncycles - c.cycles + 1) / 2);
      if (tlim > 0.0 && c.dt > 0.0) {
        const double est = (tlim - c.t) / c.dt;  // cycles left at the current dt
        if (est < 2.0 * pairs) pairs = std::max(1, (int)std::ceil(0.5 * est) + 1);
        if (ncycles >= 0) pairs = std::min(pairs, std::max(1, (ncycles - c.cycles + 1) / 2));
      }
      pairs = std::max(1, pairs);
      for (int q = 0; q < pairs; ++q) CK(cudaGraphLaunch(m->gexec[parity0], ctx->stream));
      CK(cudaMemcpyAsync(&c, m->dctl, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      if (c.stop) break;
    }
  }
  // cycles that ran: the completed ones, plus the failing one (its stages ran
  // and flipped the tables inside the graph)
  const int ran = c.cycles + (c.err_key != ULLONG_MAX ? 1 : 0);
  const long long per_cycle = 2 * (2 * G.dim + (update_two_kernels(m, G.ks, G.ke) ? 2 : 1) -
                                   (m->push_x1 ? 1 : 0)) + 2 - (use_flux_xy(m, 1) ? 1 : 0) -
                              (use_flux_xy(m, 2) ? 1 : 0);
  m->times.kernel_launches += per_cycle * ran;
  if (ran & 1) {  // the state is in the other table after an odd number of cycles
    std::swap(m->hblk, m->hblk_alt);
    std::swap(m->dblk, m->dblk_alt);
    m->parity ^= 1;
  }
  if (cycles_done) *cycles_done = c.cycles;
  *t = c.t;
  *dt = c.dt;
  pmhd_status s{};
  s.k = s.j = s.i = -1;
  if (c.err_key != ULLONG_MAX) {
    s.code = PMHD_ERR_UNPHYSICAL;
    s.stage = c.err_stage;
    s.floor_count = (long long)c.err_floors;
    decode_key(G, c.err_key, &s);
    if (st) *st = s;
    ctx->err = "unphysical state in stage " + std::to_string(s.stage);
    return PMHD_ERR_UNPHYSICAL;
  }
  if (st) {
    s.code = PMHD_OK;
    s.stage = 2;
    s.floor_count = (long long)c.floors;
    s.fallback_count = (long long)c.fallbacks;
    *st = s;
  }
  return PMHD_OK;
}

}  // namespace

int pmhd_gpu_run(pmhd_mesh* m, int ncycles, double tlim, double* t, double* dt, int* cycles_done,
                 pmhd_status* st) {
  if (!m || !t || !dt) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  if (int rc_ = drop_prefetch(m)) return rc_;  // (a graph capture must not wait on outside work)
  int rc = PMHD_OK;
  if (!(*dt > 0.0)) {
    rc = pmhd_gpu_new_dt(m, dt, st);
    if (rc) return rc;
  }
  if (graph_run_ok(m)) return graph_run(m, ncycles, tlim, t, dt, cycles_done, st);
  int n = 0;
  long long floors = 0, fallbacks = 0;
  while ((ncycles < 0 || n < ncycles) && (!(tlim > 0.0) || *t < tlim)) {
    double h = *dt;
    bool last = false;
    if (tlim > 0.0 && *t + h >= tlim) { h = tlim - *t; last = true; }
    pmhd_status s{};
    s.code = PMHD_OK;
    s.k = s.j = s.i = -1;
    double dn = 0.0;
    rc = pmhd_gpu_vl2_step(m, h, &dn, &s);
    floors += s.floor_count;
    fallbacks += s.fallback_count;
    if (rc) { if (st) *st = s; break; }
    *t = last ? tlim : *t + h;
    *dt = dn;
    ++n;
  }
  if (cycles_done) *cycles_done = n;
  // the run returns with all its device work done (the last step's deferred
  // ghost exchanges included)
  if (!rc) rc = drop_prefetch(m);
  if (!rc && cudaStreamSynchronize(m->ctx->stream) != cudaSuccess)
    rc = fail(m->ctx, PMHD_ERR_CUDA, "run: stream synchronize failed");
  if (st && rc == PMHD_OK) {
    st->code = PMHD_OK;
    st->floor_count = floors;
    st->fallback_count = fallbacks;
  }
  return rc;
}

int pmhd_gpu_diag(pmhd_mesh* m, int kind, double* out) {
  if (!m || !out) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  pmhd_ctx* ctx = m->ctx;
  const KGeom& G = m->G;
  if (int rc = drop_prefetch(m)) return rc;
  if (kind == PMHD_DIAG_DIVB_MAX) {
    int rc = reset_red(m);
    if (rc) return rc;
    launch_divb(m->dblk, G, m->dred, ctx->stream);
    rc = fetch_red(m);
    if (rc) return rc;
    out[0] = bits2d(m->hred[0].divb_bits);
    return PMHD_OK;
  }
  if (kind == PMHD_DIAG_SUMS) {
    const int nrow = (G.ke - G.ks) * (G.je - G.js);
    std::vector<double> rows(size_t(G.nb) * 5 * nrow);
    launch_row_sums(m->dblk, G, m->drows, ctx->stream);
    CK(cudaMemcpyAsync(rows.data(), m->drows, rows.size() * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int v = 0; v < 5; ++v) out[v] = 0.0;
    // blocks in gid order (oracle order); rows in (k, j) order
    std::vector<int> order(G.nb);
    for (int b = 0; b < G.nb; ++b) order[b] = b;
    for (int a = 0; a < G.nb; ++a)
      for (int c = a + 1; c < G.nb; ++c)
        if (m->gids[order[c]] < m->gids[order[a]]) std::swap(order[a], order[c]);
    for (int q = 0; q < G.nb; ++q) {
      const int b = order[q];
      for (int v = 0; v < 5; ++v) {
        double s = 0.0;
        const double* r = rows.data() + (size_t(b) * 5 + v) * nrow;
        for (int n = 0; n < nrow; ++n) s += r[n];
        out[v] += s;
      }
    }
    return PMHD_OK;
  }
  return fail(ctx, PMHD_ERR_INPUT, "unknown diagnostic");
}

//------------------------------------------------------------- multi-rank pieces
namespace {
// Ghost range [q0, q1) along dir that side r (0 lower, 1 upper) receives for
// array v (0..4 cells, 5..7 faces); same as the oracle's recv_range.
void recv_range(const KGeom& G, int dir, int r, int v, int* q0, int* q1) {
  const int ng = G.ng, s = G.ng, e = s + G.mb[dir];
  const bool normal = (v == 5 + dir);
  if (r == 0) { *q0 = 0; *q1 = normal ? s + 1 : ng; }
  else { *q0 = normal ? e + 1 : e; *q1 = e + ng + (normal ? 1 : 0); }
}
// Slab of block-side `side`: send=true -> what this block sends to that
// neighbour; send=false -> the ghosts it receives from it.
HaloSlab make_slab(const KGeom& G, int dir, int side, bool send) {
  HaloSlab sl;
  const int r = send ? 1 - side : side;
  const int sh = send ? ((r == 0) ? G.mb[dir] : -G.mb[dir]) : 0;
  long long off = 0;
  for (int v = 0; v < 8; ++v) {
    const int ext[3] = {G.n1 + (v == 5), G.n2 + (v == 6), G.n3 + (v == 7)};
    int q0, q1;
    recv_range(G, dir, r, v, &q0, &q1);
    for (int a = 0; a < 3; ++a) {
      sl.org[v][a] = (a == dir) ? q0 + sh : 0;
      sl.ext[v][a] = (a == dir) ? q1 - q0 : ext[a];
    }
    sl.off[v] = off;
    off += (long long)sl.ext[v][0] * sl.ext[v][1] * sl.ext[v][2];
  }
  sl.off[8] = off;
  return sl;
}
}  // namespace

int pmhd_gpu_stage_compute(pmhd_mesh* m, int stage, double dt, double* dt_next, pmhd_status* st) {
  if (!m) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  if (stage != 1 && stage != 2) return fail(m->ctx, PMHD_ERR_INPUT, "stage must be 1 or 2");
  if (m->async_ops) {  // reductions of both stages are checked after stage 2
    int rc = (stage == 1) ? reset_red(m) : PMHD_OK;
    if (!rc) rc = enqueue_stage(m, stage, dt, false);
    if (rc) return rc;
    if (stage == 1) {
      if (st) { std::memset(st, 0, sizeof(*st)); st->k = st->j = st->i = -1; st->stage = 1; }
      return PMHD_OK;
    }
    return finish(m, 1, 2, dt_next, st);
  }
  // a prefetched stage already accumulates into its reduction slot (reset by
  // the previous stage_compute), so it is not reset again
  int rc = (m->prefetched == stage) ? PMHD_OK : reset_red(m);
  if (!rc) rc = enqueue_stage(m, stage, dt, false);
  if (rc) return rc;
  return finish(m, stage, stage, stage == 2 ? dt_next : nullptr, st);
}

int pmhd_gpu_stage_prefetch(pmhd_mesh* m, int stage, double dt) {
  if (!m) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  if (stage != 2) return fail(m->ctx, PMHD_ERR_INPUT, "only stage 2 can be prefetched");
  if (!can_prefetch(m)) return PMHD_OK;  // stage_compute then runs every tile
  pmhd_ctx* ctx = m->ctx;
  if (m->prefetched) CK(cudaStreamWaitEvent(ctx->stream, m->ev_pre[1], 0));
  return prefetch_stage(m, stage, dt);
}

int pmhd_gpu_drive_begin(pmhd_mesh* m, int nmode, const int* k, const double* c, const double* s,
                         const double* const* cos_tab, const double* const* sin_tab, double* sums) {
  if (!m || nmode < 0 || nmode > 64 || (nmode > 0 && (!k || !c || !s)) || !cos_tab || !sin_tab || !sums)
    return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  pmhd_ctx* ctx = m->ctx;
  const KGeom& G = m->G;
  if (int rc = drop_prefetch(m)) return rc;
  if (!m->drive_tab) {
    const size_t tab = 2 * 5 * size_t(G.nx[0] + G.nx[1] + G.nx[2]);
    const size_t rows = size_t(G.nb) * (G.ke - G.ks) * ((G.je - G.js) + 1) * 4;  // rows + planes
    CK(cudaMalloc(&m->drive_tab, tab * sizeof(double)));
    CK(cudaMalloc(&m->drive_rows, rows * sizeof(double)));
    CK(cudaMalloc(&m->drive_sums, size_t(G.nb) * 4 * sizeof(double)));
  }
  DriveTabs& T = m->drive;
  T.n = nmode;
  for (int q = 0; q < nmode; ++q)
    for (int a = 0; a < 3; ++a) {
      T.k[q][a] = k[3 * q + a];
      T.c[q][a] = c[3 * q + a];
      T.s[q][a] = s[3 * q + a];
    }
  double* p = m->drive_tab;
  for (int a = 0; a < 3; ++a) {
    const size_t n = 5 * size_t(G.nx[a]);
    CK(cudaMemcpyAsync(p, cos_tab[a], n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    T.ct[a] = p;
    p += n;
    CK(cudaMemcpyAsync(p, sin_tab[a], n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    T.st[a] = p;
    p += n;
  }
  launch_drive_dv(m->dblk, G, T, ctx->stream);
  const double zero[3] = {0.0, 0.0, 0.0};
  launch_drive_sums(m->dblk, G, 0, zero, m->drive_rows, m->drive_sums, ctx->stream);
  m->times.kernel_launches += 4;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(sums, m->drive_sums, size_t(G.nb) * 4 * sizeof(double), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return PMHD_OK;
}

int pmhd_gpu_drive_energy(pmhd_mesh* m, const double* mean, double* sums) {
  if (!m || !mean || !sums || !m->drive_tab) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  pmhd_ctx* ctx = m->ctx;
  if (int rc = drop_prefetch(m)) return rc;
  launch_drive_sums(m->dblk, m->G, 1, mean, m->drive_rows, m->drive_sums, ctx->stream);
  m->times.kernel_launches += 3;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(sums, m->drive_sums, size_t(m->G.nb) * 4 * sizeof(double), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return PMHD_OK;
}

int pmhd_gpu_drive_apply(pmhd_mesh* m, const double* mean, double scale) {
  if (!m || !mean || !m->drive_tab) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  pmhd_ctx* ctx = m->ctx;
  if (int rc = drop_prefetch(m)) return rc;
  launch_drive_apply(m->dblk, m->G, mean, scale, ctx->stream);
  launch_exchange(m->dblk, m->G, 0, ctx->stream);
  m->times.kernel_launches += 1 + m->G.dim;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return PMHD_OK;
}

int pmhd_gpu_slab(const pmhd_mesh* m, void** base, void* ipc_handle) {
  if (!m || !base) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  *base = m->slab;
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    pmhd_ctx* ctx = m->ctx;
    CK(cudaIpcGetMemHandle(&h, m->slab));
    std::memcpy(ipc_handle, &h, sizeof(h));
  }
  return PMHD_OK;
}

int pmhd_gpu_ipc_open(pmhd_ctx* ctx, const void* ipc_handle, void** base) {
  if (!ctx || !ipc_handle || !base) return PMHD_ERR_INPUT;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, sizeof(h));
  CK(cudaSetDevice(ctx->device));
  CK(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  return PMHD_OK;
}

int pmhd_gpu_ipc_close(pmhd_ctx* ctx, void* base) {
  if (!ctx || !base) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(ctx)) return rc_;
  CK(cudaIpcCloseMemHandle(base));
  return PMHD_OK;
}

int pmhd_gpu_peer_attach(pmhd_mesh* m, int nranks, const int* owner_of_gid, void* const* rank_base) {
  if (!m || nranks < 1 || !owner_of_gid || !rank_base) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  pmhd_ctx* ctx = m->ctx;
  const KGeom& G = m->G;
  const pmhd_mesh_desc& d = m->desc;
  const int nb[3] = {d.nx[0] / d.mb[0], d.nx[1] / d.mb[1], d.nx[2] / d.mb[2]};
  const int ntot = nb[0] * nb[1] * nb[2];
  for (size_t b = 1; b < m->gids.size(); ++b)
    if (m->gids[b] < m->gids[b - 1]) return fail(ctx, PMHD_ERR_INPUT, "peer_attach needs gids in ascending order");
  // a rank's blocks sit in its slab in ascending gid order
  std::vector<int> slot(ntot, -1), count(nranks, 0);
  for (int g = 0; g < ntot; ++g) {
    const int r = owner_of_gid[g];
    if (r < 0 || r >= nranks) return fail(ctx, PMHD_ERR_INPUT, "owner out of range");
    slot[g] = count[r]++;
  }
  for (std::vector<DevBlock>* tab : {&m->hblk, &m->hblk_alt})
    for (int b = 0; b < G.nb; ++b) {
      DevBlock& B = (*tab)[b];
      const int gid = m->gids[b];
      const int c0[3] = {gid % nb[0], (gid / nb[0]) % nb[1], gid / (nb[0] * nb[1])};
      for (int a = 0; a < 3; ++a)
        for (int side = 0; side < 2; ++side) {
          B.rbase[a][side] = nullptr;
          if (a >= G.dim || B.nbr[a][side] >= 0) continue;  // local neighbour
          int c[3] = {c0[0], c0[1], c0[2]};
          c[a] = (c[a] + (side ? 1 : -1) + nb[a]) % nb[a];
          const int ng = (c[2] * nb[1] + c[1]) * nb[0] + c[0];
          const char* rb = static_cast<const char*>(rank_base[owner_of_gid[ng]]);
          if (!rb) continue;  // no mapping: halo pack / unpack serves this face
          B.rbase[a][side] = rb + size_t(slot[ng]) * m->per_block * sizeof(double);
        }
    }
  CK(cudaMemcpy(m->dblk, m->hblk.data(), sizeof(DevBlock) * G.nb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(m->dblk_alt, m->hblk_alt.data(), sizeof(DevBlock) * G.nb, cudaMemcpyHostToDevice));
  for (auto& g : m->gexec) if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  return PMHD_OK;
}

int pmhd_gpu_set_async(pmhd_mesh* m, int on) {
  if (!m) return PMHD_ERR_INPUT;
  m->async_ops = on != 0;
  return PMHD_OK;
}

int pmhd_gpu_exchange_dir(pmhd_mesh* m, int dir, int half) {
  if (!m || dir < 0 || dir >= m->G.dim) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  pmhd_ctx* ctx = m->ctx;
  launch_exchange_dir(m->dblk, m->G, half ? 1 : 0, dir, ctx->stream);
  m->times.kernel_launches += 1;
  CK(cudaGetLastError());
  if (!m->async_ops) CK(cudaStreamSynchronize(ctx->stream));
  return PMHD_OK;
}

int pmhd_gpu_halo_count(const pmhd_mesh* m, int dir, int side, long long* n) {
  if (!m || !n || dir < 0 || dir >= m->G.dim || side < 0 || side > 1) return PMHD_ERR_INPUT;
  *n = make_slab(m->G, dir, side, false).off[8];
  return PMHD_OK;
}

static int halo_xfer(pmhd_mesh* m, int gid, int dir, int side, int half, double* dev_buf, bool pack) {
  if (!m || !dev_buf || dir < 0 || dir >= m->G.dim || side < 0 || side > 1) return PMHD_ERR_INPUT;
  if (int rc_ = use_device(m->ctx)) return rc_;
  pmhd_ctx* ctx = m->ctx;
  const int b = local_index(m, gid);
  if (b < 0) return fail(ctx, PMHD_ERR_INPUT, "block not local");
  const HaloSlab sl = make_slab(m->G, dir, side, pack);
  double* const* arrays = &m->dblk[b].st[half ? 1 : 0][0];  // device address of the 8 pointers
  launch_halo_copy(arrays, m->G, sl, dev_buf, pack ? 1 : 0, ctx->stream);
  m->times.kernel_launches += 1;
  CK(cudaGetLastError());
  if (!m->async_ops) CK(cudaStreamSynchronize(ctx->stream));
  return PMHD_OK;
}

int pmhd_gpu_halo_pack(pmhd_mesh* m, int gid, int dir, int side, int half, double* dev_buf) {
  return halo_xfer(m, gid, dir, side, half, dev_buf, true);
}

int pmhd_gpu_halo_unpack(pmhd_mesh* m, int gid, int dir, int side, int half, const double* dev_buf) {
  return halo_xfer(m, gid, dir, side, half, const_cast<double*>(dev_buf), false);
}

int pmhd_gpu_set_profiling(pmhd_mesh* m, int on) {
  if (!m) return PMHD_ERR_INPUT;
  if (on < 0 || on > 2) return fail(m->ctx, PMHD_ERR_INPUT, "profiling mode must be 0, 1 or 2");
  m->prof = on != 0;
  m->ph.prof = (on == 1) ? 1 : 0;  // 2: events only, product kernels
  return PMHD_OK;
}

int pmhd_gpu_region_times(pmhd_mesh* m, pmhd_region_times* out, int reset) {
  if (!m) return PMHD_ERR_INPUT;
  if (out) *out = m->times;
  if (reset) std::memset(&m->times, 0, sizeof(m->times));
  return PMHD_OK;
}

}  // extern "C"

extern "C" void* pmhd_gpu_stream(const pmhd_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
