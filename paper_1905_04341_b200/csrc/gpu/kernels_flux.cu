// kernels_flux.cu -- fused (cons_to_prim + reconstruction + Riemann) face-flux
// kernel, one launch per direction per stage over all MeshBlocks.
//
// Replaces the reference ops plm_reconstruct + riemann (the
// "reconstruct" and "riemann" regions of SPEC.md:527) and the stage-input
// cons_to_prim for the cells each tile touches.
//
// Tiling: a CTA of 128 threads owns 32 x 8 faces: 32 consecutive faces along
// i (coalesced HBM rows) times 8 positions along the second tile axis (j for
// x1/x2 faces, k for x3 faces) in one plane (x1/x2) or one row (x3).
//  phase 1  the stencil cells of the tile (36 x 8 for x1, 32 x 11 for x2/x3)
//           are loaded once with coalesced loads and converted to the 7
//           rotated primitives in shared memory;
//  phase 2  each cell's PLM slope is formed ONCE per variable and the two
//           reconstructed interface values q -/+ dq/2 replace it in shared
//           memory (stage 2 only; stage 1 is donor cell);
//  phase 3  each thread solves 2 faces from shared memory (no HBM waits).
// The last direction's kernel also writes the cell-centred E = -v x B of the
// box the fused update kernel needs (cells [is-1,ie] x [js-1,je] x [ks-1,ke]),
// so that kernel does not redo cons_to_prim.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"

namespace pmhd_gpu {

namespace {

#ifndef PMHD_FLUX_T_FX
#define PMHD_FLUX_T_FX 16  // x2 / x3 tiles: faces along i
#endif
#ifndef PMHD_FLUX_STCS
#define PMHD_FLUX_STCS 1  // streaming (evict-first) stores of the face data (+0.3 %)
#endif
#ifndef PMHD_P1_BATCH
#define PMHD_P1_BATCH 3  // stencil cells whose loads are batched per thread
#endif
#ifndef PMHD_FLUX_STAGE1_SKIP
#define PMHD_FLUX_STAGE1_SKIP 1  // stage-1 tiles skip the outer PLM stencil cells
#endif
#ifndef PMHD_FLUX_X1_FX
#define PMHD_FLUX_X1_FX 32  // x1 tiles: faces along i
#endif
constexpr int NTHR = 128;
#ifndef PMHD_FLUX_CPASYNC
#define PMHD_FLUX_CPASYNC 0  // 1: phase-1 stencil loads as cp.async into shared memory
#endif
#if PMHD_FLUX_CPASYNC
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
#endif
#ifndef PMHD_FLUX_FACE_UNROLL
#define PMHD_FLUX_FACE_UNROLL 1  // 2: both faces of a thread in one unrolled body
#endif
constexpr int kFaceUnroll = PMHD_FLUX_FACE_UNROLL;
#ifndef PMHD_FLUX_SMEMW
#define PMHD_FLUX_SMEMW 1
#endif
// Resident CTAs per SM the register budget is sized for: Roe needs ~130
// registers (4 CTAs); HLLD with shared-memory side states (SmemW) and HLLE
// fit 96 (5 CTAs, 20 warps; shared memory allows 5 for the 39 KB x2/x3 tiles).
#ifndef PMHD_FLUX_MINB
#define PMHD_FLUX_MINB 5
#endif
#ifndef PMHD_FLUX_MINB_ROE
#define PMHD_FLUX_MINB_ROE 4
#endif
template <int RS>
struct FluxMinB {
  static constexpr int value = (RS == PMHD_RIEMANN_ROE) ? PMHD_FLUX_MINB_ROE : PMHD_FLUX_MINB;
};

template <int DIR>
struct TileShape {
  // faces per tile: 32 x 8 for x1 (halo along i: 36 x 8 cells); 16 x 16 for
  // x2 / x3 (halo along the second axis: 16 x 19 cells, 1.19 cells per face
  // instead of 1.375 for 32 x 8, and 34 KB of shared memory instead of 39 KB)
  static constexpr int FX = (DIR == 0) ? PMHD_FLUX_X1_FX : PMHD_FLUX_T_FX;  // faces along i
  static constexpr int FS = 256 / FX;                          // faces along the 2nd axis
  static constexpr int NCOL = (DIR == 0) ? FX + 4 : FX;  // cells along i
  static constexpr int NROW = (DIR == 0) ? FS : FS + 3;  // cells along the 2nd axis
  static constexpr int NCELL = NCOL * NROW;
  static constexpr int DC = (DIR == 0) ? 1 : NCOL;       // stencil stride in the tile
  static constexpr int PER = (NCELL + NTHR - 1) / NTHR;  // cells per thread
};

// Lab index of the 7 rotated variables (d, vn, vt1, vt2, p, bt1, bt2).
template <int DIR>
__device__ __forceinline__ int rot_var(int n) {
  constexpr int V[3][7] = {{0, 1, 2, 3, 4, 6, 7}, {0, 2, 3, 1, 4, 7, 5}, {0, 3, 1, 2, 4, 5, 6}};
  return V[DIR][n];
}

// Owned-face reuse (launch flag `reuse`; every neighbour of every block on
// this rank, diagonals included, is local and the blocks form a regular
// periodic grid).  The update kernel reads face data on the block's halo
// positions too: the upper normal face e of each direction and the
// transverse faces at s-1 and e.  Each of those equals, bit for bit, a face
// some block computes inside its own range [s, e) -- the ghost cells are
// exact copies, so the stencils are the same values -- so tiles cover only
// [s, e) on every axis and a face on the rim of that range is also stored
// at the halo positions that image it: coordinate s -> the lower neighbour's
// e (shift +mb), coordinate e-1 -> the upper neighbour's s-1 (shift -mb; not
// along the face's own normal axis, which has no s-1 face), and every
// combination of those across axes (edge and corner images).  The same for
// the cell-centred E the last direction writes (cells s-1 and e of the two
// tile axes in the plane).  At 256^3 this removes the partial tiles of the
// extended ranges (x1: 257 faces in 9 tiles of 32, x2/x3: 258 in 17 of 16),
// 12-15 % of the flux CTAs; with 64^3 blocks about a third.
// axes: bit a set = axis a may image; normal: the axis that images its s
// only (-1: none).  ci/cj/ck: the value's coordinates.  SEL 0..2: the face
// data of that direction (vals in rotated order, stored to the lab-order
// arrays); SEL 3: the cell-centred E (3 values).  Fully unrolled, so the
// bookkeeping stays in registers.
template <int SEL>
__device__ __forceinline__ void rim_images(const DevBlock* __restrict__ blks, int b, const KGeom& G, int axes,
                                           int normal, int ci, int cj, int ck, int id, const double* vals) {
  constexpr int NV = (SEL < 3) ? 8 : 3;
  const int c[3] = {ci, cj, ck}, s[3] = {G.is, G.js, G.ks}, e[3] = {G.ie, G.je, G.ke};
  const int st[3] = {1, G.sx, G.sy};
  int side[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    side[a] = -1;
    if ((axes >> a) & 1) {
      if (c[a] == s[a]) side[a] = 0;
      else if (c[a] == e[a] - 1 && a != normal) side[a] = 1;
    }
  }
  if (side[0] < 0 && side[1] < 0 && side[2] < 0) return;
#pragma unroll
  for (int msk = 1; msk < 8; ++msk) {
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (((msk >> a) & 1) && side[a] < 0) ok = false;
    if (!ok) continue;
    int t = b, off = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if ((msk >> a) & 1) {
        t = blks[t].nbr[a][side[a]];
        off += (side[a] == 0 ? G.mb[a] : -G.mb[a]) * st[a];
      }
    const DevBlock& TB = blks[t];
    PMHD_CHECK_ID(G, id + off);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double* dst;
      if constexpr (SEL < 3) dst = TB.fx[SEL][(v >= 1 && v <= 3) ? rot_var<SEL>(v) : v];
      else dst = TB.ec[v];
      __stcs(dst + id + off, vals[v]);
    }
  }
}

// MODE: 0 product, 1 region profiling (phase clocks), 2 graph-replayed cycle
// (coefficient and skip flag read from the device copy kd)
template <int DIR, int RS, int MODE>
__global__ void __launch_bounds__(NTHR, FluxMinB<RS>::value)
k_flux_fused(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, int sel, int plm, double c1024_arg,
             const KStage* __restrict__ kd, int stage, DevRed* red, int write_ec, int f_i0, int f_i1,
             int f_s0, int f_s1, int f_t0, int f_t1, int ty0, int region, int reuse) {
  constexpr bool PROF = (MODE == 1);
  if (MODE == 2 && kd->skip) return;  // replayed cycle past the end of the run: no loads either
  using TS = TileShape<DIR>;
  __shared__ double sw[7][TS::NCELL];  // primitives; after phase 2: q - dq/2 (low-face value)
  __shared__ double sp[7][TS::NCELL];  // after phase 2: q + dq/2 (high-face value)
  __shared__ long long tph[3];          // profiling: phase start clocks (thread 0)
  if (PROF && threadIdx.x == 0) tph[0] = clock64();

  const int nt = f_t1 - f_t0;
  const int b = blockIdx.z / nt;
  const int t3 = f_t0 + (int)(blockIdx.z % nt);   // k for x1/x2, j for x3
  constexpr int FX = TS::FX, FS = TS::FS;
  const int fi0 = f_i0 + blockIdx.x * FX;          // first face along i
  const int fs0 = f_s0 + (ty0 + blockIdx.y) * FS;  // first face along the 2nd axis
  const DevBlock& B = blks[b];
  double* const* S = B.st[sel];
  // owned-face reuse: does this tile hold a face (or an E cell) on the rim
  // of the owned range, i.e. anything with halo images?  (per-tile test;
  // the per-face test in rim_images then runs on rim tiles only)
  bool rim = false;
  if (reuse) {
    const int s1 = fs0, e1 = fs0 + FS - 1;  // the tile's second-axis range
    const int fi1 = fi0 + FX - 1;
    if (DIR == 0) rim = fi0 <= G.is || s1 <= G.js || e1 >= G.je - 1 || (G.dim == 3 && (t3 <= G.ks || t3 >= G.ke - 1));
    else if (DIR == 1) rim = fi0 <= G.is || fi1 >= G.ie - 1 || s1 <= G.js || (G.dim == 3 && (t3 <= G.ks || t3 >= G.ke - 1));
    else rim = fi0 <= G.is || fi1 >= G.ie - 1 || t3 <= G.js || t3 >= G.je - 1 || s1 <= G.ks;
  }
  if (region != 0) {
    // region 1: only tiles whose stencil (cells and the faces their Bcc
    // averages read) avoids everything the ghost exchange writes -- ghost
    // cells and the lower normal face s of each axis; region 2: the rest.
    // Lets the interior tiles of a stage run while the exchange of the
    // previous stage is in flight.
    int c0[3], c1[3];  // inclusive cell box (i, j, k) of the tile's stencil
    if (DIR == 0) { c0[0] = fi0 - 2; c1[0] = fi0 + FX + 1; c0[1] = fs0; c1[1] = fs0 + FS - 1; c0[2] = c1[2] = t3; }
    else if (DIR == 1) { c0[0] = fi0; c1[0] = fi0 + FX - 1; c0[1] = fs0 - 2; c1[1] = fs0 + FS + 1; c0[2] = c1[2] = t3; }
    else { c0[0] = fi0; c1[0] = fi0 + FX - 1; c0[2] = fs0 - 2; c1[2] = fs0 + FS + 1; c0[1] = c1[1] = t3; }
    bool inner = c0[0] >= G.is + 1 && c1[0] <= G.ie - 1 && c0[1] >= G.js + 1 && c1[1] <= G.je - 1;
    if (G.dim == 3) inner = inner && c0[2] >= G.ks + 1 && c1[2] <= G.ke - 1;
    if (inner != (region == 1)) return;
  }

  // ---- phase 1: load + cons_to_prim of the stencil cells into smem --------
  // tile cell c -> its (k, j, i); false outside the block array
  auto cell_ijk = [&](int c, int& i, int& j, int& k) {
    const int col = c % TS::NCOL, row = c / TS::NCOL;
    if (DIR == 0) { i = fi0 - 2 + col; j = fs0 + row; k = t3; }
    else if (DIR == 1) { i = fi0 + col; j = fs0 - 2 + row; k = t3; }
    else { i = fi0 + col; k = fs0 - 2 + row; j = t3; }
    // donor cell (stage 1) reads only the two cells adjacent to each face:
    // the outer PLM stencil positions (x1: columns 0, FX+2, FX+3; x2 / x3:
    // rows 0, FS+2) are skipped -- except row FS+2 when this tile owns that
    // cell-centred E row (write_ec, owned ranges, last tile)
    if (PMHD_FLUX_STAGE1_SKIP && !plm) {
      const int pos = (DIR == 0) ? col : row;
      if (pos == 0 || pos >= ((DIR == 0) ? FX + 2 : FS + 2)) {
        const bool ec_row = (DIR != 0) && write_ec && reuse && pos == FS + 2 && fs0 + FS == f_s1;
        if (!ec_row) return false;
      }
    }
    return c < TS::NCELL && i >= 0 && i < G.n1 && j >= 0 && j < G.n2 && k >= 0 && k < G.n3;
  };
  // cons_to_prim of tile cell c (block index id) from its 11 raw values (5
  // conserved, then the face pairs b1f, b2f, b3f); writes the 7 rotated
  // primitives to sw[.][c] (and the cell-centred E where this tile owns it)
  auto finish = [&](int c, int id, const double* ub) {
    double u[5], bc[3], w[8];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = ub[v];
    bc[0] = 0.5 * (ub[5] + ub[6]);
    bc[1] = 0.5 * (ub[7] + ub[8]);
    bc[2] = 0.5 * (ub[9] + ub[10]);
    const int fl = cons_to_prim(u, bc, ph, w, false);
    int i, j, k;
    cell_ijk(c, i, j, k);
    if ((fl & 4) && k >= G.ks && k < G.ke && j >= G.js && j < G.je && i >= G.is && i < G.ie) {
      const long long gi = (long long)B.c[0] * G.mb[0] + (i - G.is);
      const long long gj = (long long)B.c[1] * G.mb[1] + (j - G.js);
      const long long gk = (G.dim == 3) ? (long long)B.c[2] * G.mb[2] + (k - G.ks) : 0;
      atomicMin(&red[stage].bad_key, (unsigned long long)((gk * G.nx[1] + gj) * G.nx[0] + gi));
    }
    if (DIR != 0 && write_ec) {
      // cells of this tile's own face rows [fs0, fs0+8) clipped to the face
      // range, plus the row below the block's first face row
      const int s = (DIR == 2) ? k : j;
      // (owned face ranges: also the row above the last face row, which the
      // extended ranges covered as a face row of their own)
      const bool own = (s >= fs0 && s < fs0 + FS && s < f_s1) || (fs0 == f_s0 && s == f_s0 - 1) ||
                       (reuse && s == f_s1 && fs0 + FS >= f_s1);
      if (own && i >= f_i0 && i < f_i1) {
        const double ev[3] = {w[3] * w[6] - w[2] * w[7], w[1] * w[7] - w[3] * w[5], w[2] * w[5] - w[1] * w[6]};
        B.ec[0][id] = ev[0];
        B.ec[1][id] = ev[1];
        B.ec[2][id] = ev[2];
        if (rim) {  // images on the neighbours' halo columns / rows of the plane
          rim_images<3>(blks, b, G, (DIR == 2) ? 3 : 1, -1, i, j, k, id, ev);
        }
      }
    }
#pragma unroll
    for (int n = 0; n < 7; ++n) sw[n][c] = w[rot_var<DIR>(n)];
  };
#if PMHD_FLUX_CPASYNC
  {
    // every raw value of this thread's cells in flight at once without
    // registers: cp.async into shared memory (conserved -> sp[0..4][c],
    // faces -> sw[0..5][c]; both are free until phase 1 writes sw[.][c] of
    // the same cell, from the same thread)
    int cid[TS::PER];
#pragma unroll
    for (int p = 0; p < TS::PER; ++p) {
      cid[p] = -1;
      const int c = threadIdx.x + p * NTHR;
      int i, j, k;
      if (cell_ijk(c, i, j, k)) {
        const int id = G.idx(k, j, i);
        cid[p] = id;
#pragma unroll
        for (int v = 0; v < 5; ++v) cp_async8(&sp[v][c], S[v] + id);
        cp_async8(&sw[0][c], S[5] + id);
        cp_async8(&sw[1][c], S[5] + id + 1);
        cp_async8(&sw[2][c], S[6] + id);
        cp_async8(&sw[3][c], S[6] + id + G.sx);
        cp_async8(&sw[4][c], S[7] + id);
        cp_async8(&sw[5][c], S[7] + id + G.sy);
      }
    }
    cp_async_wait_all();
#pragma unroll
    for (int p = 0; p < TS::PER; ++p) {
      if (cid[p] < 0) continue;
      const int c = threadIdx.x + p * NTHR;
      double ub[11];
#pragma unroll
      for (int v = 0; v < 5; ++v) ub[v] = sp[v][c];
#pragma unroll
      for (int q = 0; q < 6; ++q) ub[5 + q] = sw[q][c];
      finish(c, cid[p], ub);
    }
  }
#else
  // The loads of PMHD_P1_BATCH cells are issued before any is consumed
  // (memory-level parallelism: up to BATCH x 11 loads in flight per thread).
  constexpr int NB = (PMHD_P1_BATCH < TS::PER) ? PMHD_P1_BATCH : TS::PER;
#pragma unroll
  for (int p0 = 0; p0 < TS::PER; p0 += NB) {
    double ub[NB][11];
    int cid[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int p = p0 + q;
      cid[q] = -1;
      if (p >= TS::PER) continue;
      const int c = threadIdx.x + p * NTHR;
      int i, j, k;
      if (cell_ijk(c, i, j, k)) {
        const int id = G.idx(k, j, i);
        PMHD_CHECK_ID(G, id + G.sy);
        cid[q] = id;
#pragma unroll
        for (int v = 0; v < 5; ++v) ub[q][v] = __ldg(S[v] + id);
        ub[q][5] = __ldg(S[5] + id);
        ub[q][6] = __ldg(S[5] + id + 1);
        ub[q][7] = __ldg(S[6] + id);
        ub[q][8] = __ldg(S[6] + id + G.sx);
        ub[q][9] = __ldg(S[7] + id);
        ub[q][10] = __ldg(S[7] + id + G.sy);
      }
    }
#pragma unroll
    for (int q = 0; q < NB; ++q)
      if (cid[q] >= 0) finish(threadIdx.x + (p0 + q) * NTHR, cid[q], ub[q]);
  }
#endif
  __syncthreads();
  if (PROF && threadIdx.x == 0) tph[1] = clock64();

  // ---- phase 2: per-cell reconstruction, one variable at a time ------------
#ifdef PMHD_DIAG_NO_PLM  // diagnostic build only: donor-cell states in stage 2 too
  plm = 0;
#endif
  if (plm) {
    constexpr int LEN = (DIR == 0) ? TS::NCOL : TS::NROW;
    // which of this thread's cells have both stencil neighbours in the tile
    // (evaluated once, not per variable)
    unsigned vmask = 0;
#pragma unroll
    for (int p = 0; p < TS::PER; ++p) {
      const int c = threadIdx.x + p * NTHR;
      const int pos = (DIR == 0) ? c % TS::NCOL : c / TS::NCOL;
      if (c < TS::NCELL && pos >= 1 && pos <= LEN - 2) vmask |= 1u << p;
    }
#pragma unroll 1
    for (int n = 0; n < 7; ++n) {
      double lo[TS::PER], hi[TS::PER];
      double* const q = &sw[n][threadIdx.x];
#pragma unroll
      for (int p = 0; p < TS::PER; ++p) {
        if (vmask & (1u << p)) {
          const double q0 = q[p * NTHR];
          const double hdq = plm_half_slope(q[p * NTHR - TS::DC], q0, q[p * NTHR + TS::DC], ph.limiter);
          hi[p] = q0 + hdq;  // wL of the face above (oracle: qm1 + 0.5*slope)
          lo[p] = q0 - hdq;  // wR of the face below (oracle: q0 - 0.5*slope)
        }
      }
      __syncthreads();  // all reads of sw[n] done before it is overwritten
#pragma unroll
      for (int p = 0; p < TS::PER; ++p) {
        if (vmask & (1u << p)) {
          q[p * NTHR] = lo[p];
          sp[n][threadIdx.x + p * NTHR] = hi[p];
        }
      }
    }
    __syncthreads();
  }

  if (PROF && threadIdx.x == 0) tph[2] = clock64();

  // ---- phase 3: two faces per thread ---------------------------------------
  const int fc = threadIdx.x % FX;
  const double c1024 = (MODE == 2) ? kd->c1024[DIR] : c1024_arg;
  const double* const wsrc = plm ? &sp[0][0] : &sw[0][0];  // low-side cell's high-face value
#pragma unroll kFaceUnroll
  for (int h = 0; h < 2; ++h) {
    const int fr = threadIdx.x / FX + (NTHR / FX) * h;
    const int fi = fi0 + fc, fs = fs0 + fr;
    if (fi >= f_i1 || fs >= f_s1) continue;
    const int cl = fr * TS::NCOL + fc + TS::DC;  // cell on the low side of the face
    const int ch = cl + TS::DC;                  // cell on the high side
    int i, j, k;
    if (DIR == 0) { i = fi; j = fs; k = t3; }
    else if (DIR == 1) { i = fi; j = fs; k = t3; }
    else { i = fi; k = fs; j = t3; }
    const int id = G.idx(k, j, i);
    PMHD_CHECK_ID(G, id);
    const double bn = __ldg(S[5 + DIR] + id);
    double out[8];
    int fb;
    if constexpr (PMHD_FLUX_SMEMW && (RS == PMHD_RIEMANN_HLLD || RS == PMHD_RIEMANN_ROE)) {
      const SmemW wl{wsrc + cl, TS::NCELL}, wr{&sw[0][0] + ch, TS::NCELL};
      fb = face_solve<RS>(wl, wr, bn, ph, c1024, out);
    } else {
      double wl[7], wr[7];
#pragma unroll
      for (int n = 0; n < 7; ++n) {
        wl[n] = wsrc[n * TS::NCELL + cl];
        wr[n] = sw[n][ch];
      }
      fb = face_solve<RS>(wl, wr, bn, ph, c1024, out);
    }
    if (fb)
      atomicAdd(&red[stage].fallback_count, 1ULL);
    double* const* F = B.fx[DIR];
#ifdef PMHD_DIAG_NO_FACE_STORES  // diagnostic build only: skip the face-data stores
    if (out[0] == 12345.678) F[0][id] = out[1];  // (keeps the solve live)
    continue;
#endif
#if PMHD_FLUX_STCS  // streaming stores: the face data is read back by the next kernel, not reused here
    __stcs(F[0] + id, out[0]);
    __stcs(F[rot_var<DIR>(1)] + id, out[1]);
    __stcs(F[rot_var<DIR>(2)] + id, out[2]);
    __stcs(F[rot_var<DIR>(3)] + id, out[3]);
    __stcs(F[4] + id, out[4]);
    __stcs(F[5] + id, out[5]);
    __stcs(F[6] + id, out[6]);
    __stcs(F[7] + id, out[7]);
#else
    F[0][id] = out[0];
    F[rot_var<DIR>(1)][id] = out[1];
    F[rot_var<DIR>(2)][id] = out[2];
    F[rot_var<DIR>(3)][id] = out[3];
    F[4][id] = out[4];
    F[5][id] = out[5];
    F[6][id] = out[6];
    F[7][id] = out[7];
#endif
    if (rim) {  // a face on the rim of the owned range: its halo images
      rim_images<DIR>(blks, b, G, (G.dim == 3) ? 7 : 3, DIR, i, j, k, id, out);
    }
  }
  if (PROF) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long t3 = clock64();
      atomicAdd(&red[stage].phase[0], (unsigned long long)(tph[1] - tph[0]));
      atomicAdd(&red[stage].phase[1], (unsigned long long)(tph[2] - tph[1]));
      atomicAdd(&red[stage].phase[2], (unsigned long long)(t3 - tph[2]));
    }
  }
}

//---------------------------------------------------------------------------
// Column-march flux kernel for the x2 and x3 faces (DIR 1: march along j,
// DIR 2: march along k; the default for them).  Their stencil runs along an axis the threads of a
// warp do not share (a warp is 32 consecutive i), so each thread owns one
// face column and walks it: per step it loads and converts ONE new cell,
// forms ONE PLM slope and solves ONE face, keeping the last three cells'
// rotated primitives and the reconstructed side states in a private slice of
// shared memory ([var][thread], conflict-free; HLLD reads its side states
// from there through SmemW as in k_flux_fused).  No thread reads another
// thread's data, so there is no __syncthreads at all, and a column segment
// of L faces converts L + 3 cells (the tile kernel: 1.19 per face), and the
// next cell's raw values are loaded one step ahead into registers, so their
// latency hides behind the current face's solve (the tile kernel cannot:
// its loads precede a CTA barrier).  Same expressions and operand order as
// k_flux_fused, so the same bits.
#ifndef PMHD_MARCH_L
#define PMHD_MARCH_L 24  // faces per column segment (measured: 16 / 24 / 32 / 48 -> 7.60 / 7.56 / 7.60 / 7.58 ms)
#endif
constexpr int MT = 128;  // threads: 32 i x 4 transverse columns
#ifndef PMHD_MARCH_PREFETCH
#define PMHD_MARCH_PREFETCH 1  // load the next cell's raw values one step ahead
#endif
#ifndef PMHD_MARCH_MINB
#define PMHD_MARCH_MINB 4  // CTAs per SM the registers are sized for (5 spills 24-32 B)
#endif
template <int RS>
struct MarchMinB {
  static constexpr int value = PMHD_MARCH_MINB ? PMHD_MARCH_MINB : FluxMinB<RS>::value;
};
template <int DIR, int RS, int MODE>
__global__ void __launch_bounds__(MT, MarchMinB<RS>::value)
k_flux_march(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, int sel, int plm, double c1024_arg,
             const KStage* __restrict__ kd, int stage, DevRed* red, int write_ec, int f_i0, int f_i1, int f_m0,
             int f_m1, int f_t0, int f_t1, int region, int reuse) {
  static_assert(DIR == 1 || DIR == 2, "column march: x2 / x3 faces");
  constexpr bool PROF = (MODE == 1);
  if (MODE == 2 && kd->skip) return;
  // private ring: P[slot][var][thread] primitives of the last 3 cells (rotated
  // order), WL[2] high-face states of the previous / this cell, WR the
  // low-face state of this cell (stage 2); stage 1 reads P directly
  __shared__ double P[3][7][MT];
  __shared__ double WL[2][7][MT];
  __shared__ double WR[7][MT];
  const int nm = (f_m1 - f_m0 + PMHD_MARCH_L - 1) / PMHD_MARCH_L;
  const int b = blockIdx.z / nm;
  const int m0 = f_m0 + (int)(blockIdx.z % nm) * PMHD_MARCH_L;
  const int m1 = min(m0 + PMHD_MARCH_L, f_m1);
  const int i = f_i0 + blockIdx.x * 32 + (threadIdx.x & 31);
  const int t = f_t0 + blockIdx.y * 4 + (threadIdx.x >> 5);
  const DevBlock& B = blks[b];
  double* const* S = B.st[sel];
  if (region != 0) {  // as k_flux_fused: region 1 = segments clear of the ghost exchange
    const int ci0 = f_i0 + blockIdx.x * 32, ct0 = f_t0 + blockIdx.y * 4;
    int c0[3], c1[3];
    c0[0] = ci0; c1[0] = ci0 + 31;
    if (DIR == 1) { c0[1] = m0 - 2; c1[1] = m1 + 1; c0[2] = ct0; c1[2] = ct0 + 3; }
    else { c0[2] = m0 - 2; c1[2] = m1 + 1; c0[1] = ct0; c1[1] = ct0 + 3; }
    bool inner = c0[0] >= G.is + 1 && c1[0] <= G.ie - 1 && c0[1] >= G.js + 1 && c1[1] <= G.je - 1;
    if (G.dim == 3) inner = inner && c0[2] >= G.ks + 1 && c1[2] <= G.ke - 1;
    if (inner != (region == 1)) return;
  }
  if (i >= f_i1 || t >= f_t1) return;  // (no barriers below)
  const int tid = threadIdx.x;
  long long tc = 0, tp = 0, tr = 0, tck = 0;  // profiling (thread 0): c2p / PLM / Riemann cycles
  auto cid = [&](int m) { return (DIR == 2) ? G.idx(m, t, i) : G.idx(t, m, i); };
  // load + cons_to_prim of the cell at march position m into ring slot sl
  // (and its cell-centred E where this segment owns it)
  auto in_range = [&](int m) { return m >= 0 && m < ((DIR == 2) ? G.n3 : G.n2); };
  // the cell's 11 raw values (5 conserved, then the face pairs)
  auto load_raw = [&](int m, double* ub) {
    if (!in_range(m)) return;
    const int id = cid(m);
    PMHD_CHECK_ID(G, id + G.sy);
#pragma unroll
    for (int v = 0; v < 5; ++v) ub[v] = __ldg(S[v] + id);
    ub[5] = __ldg(S[5] + id);
    ub[6] = __ldg(S[5] + id + 1);
    ub[7] = __ldg(S[6] + id);
    ub[8] = __ldg(S[6] + id + G.sx);
    ub[9] = __ldg(S[7] + id);
    ub[10] = __ldg(S[7] + id + G.sy);
  };
  // cons_to_prim of the cell at march position m from its raw values
  auto conv = [&](int m, int sl, const double* ub) {
    if (!in_range(m)) return;
    const int id = cid(m);
    double u[5], bc[3], w[8];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = ub[v];
    bc[0] = 0.5 * (ub[5] + ub[6]);
    bc[1] = 0.5 * (ub[7] + ub[8]);
    bc[2] = 0.5 * (ub[9] + ub[10]);
    const int fl = cons_to_prim(u, bc, ph, w, false);
    const int k = (DIR == 2) ? m : t, j = (DIR == 2) ? t : m;
    if ((fl & 4) && k >= G.ks && k < G.ke && j >= G.js && j < G.je && i >= G.is && i < G.ie) {
      const long long gi = (long long)B.c[0] * G.mb[0] + (i - G.is);
      const long long gj = (long long)B.c[1] * G.mb[1] + (j - G.js);
      const long long gk = (G.dim == 3) ? (long long)B.c[2] * G.mb[2] + (k - G.ks) : 0;
      atomicMin(&red[stage].bad_key, (unsigned long long)((gk * G.nx[1] + gj) * G.nx[0] + gi));
    }
    if (write_ec) {
      // rows [f_m0 - 1, f_m1) (+ f_m1 with owned ranges), each by one segment
      const bool own = (m >= m0 && m < m1) || (m0 == f_m0 && m == f_m0 - 1) || (reuse && m == f_m1 && m1 == f_m1);
      if (own) {
        const double ev[3] = {w[3] * w[6] - w[2] * w[7], w[1] * w[7] - w[3] * w[5], w[2] * w[5] - w[1] * w[6]};
        B.ec[0][id] = ev[0];
        B.ec[1][id] = ev[1];
        B.ec[2][id] = ev[2];
        if (reuse) rim_images<3>(blks, b, G, (DIR == 2) ? 3 : 1, -1, i, j, k, id, ev);
      }
    }
#pragma unroll
    for (int n = 0; n < 7; ++n) P[sl][n][tid] = w[rot_var<DIR>(n)];
  };
  auto cell = [&](int m, int sl) {
    double ub[11];
    load_raw(m, ub);
    conv(m, sl, ub);
  };
  const double c1024 = (MODE == 2) ? kd->c1024[DIR] : c1024_arg;
  // prologue: cells m0-2, m0-1 (donor: m0-1 is the first face's low side;
  // PLM: both feed the first slope), ring slot = position mod 3
  auto slot = [](int m) { return ((m % 3) + 3) % 3; };
  if (PROF && tid == 0) tck = clock64();
  cell(m0 - 2, slot(m0 - 2));
  cell(m0 - 1, slot(m0 - 1));
  if (plm) {
    // high-face state of cell m0-1 (slope from m0-2, m0-1, m0)
    cell(m0, slot(m0));
#pragma unroll
    for (int n = 0; n < 7; ++n) {
      const double q0 = P[slot(m0 - 1)][n][tid];
      const double hdq = plm_half_slope(P[slot(m0 - 2)][n][tid], q0, P[slot(m0)][n][tid], ph.limiter);
      WL[(m0 - 1) & 1][n][tid] = q0 + hdq;
    }
  }
  if (PROF && tid == 0) { const long long c = clock64(); tc += c - tck; tck = c; }
  // the raw values of the next cell a step converts are loaded one step
  // ahead (PMHD_MARCH_PREFETCH), so their latency hides behind the solve
  const int ahead = plm ? 1 : 0;  // step f converts cell f + ahead
  double pre[11];
  if (PMHD_MARCH_PREFETCH) load_raw(m0 + ahead, pre);
#if PMHD_MARCH_PREFETCH == 2
  double pre2[11];  // two cells ahead
  if (m0 + 1 < m1) load_raw(m0 + 1 + ahead, pre2);
#endif
  for (int f = m0; f < m1; ++f) {
    // cell f (donor) / f+1 (PLM) -- the last one the face at f needs
    if (PMHD_MARCH_PREFETCH) {
      conv(f + ahead, slot(f + ahead), pre);
#if PMHD_MARCH_PREFETCH == 2
#pragma unroll
      for (int q = 0; q < 11; ++q) pre[q] = pre2[q];
      if (f + 2 < m1) load_raw(f + 2 + ahead, pre2);
#else
      if (f + 1 < m1) load_raw(f + 1 + ahead, pre);
#endif
    } else {
      cell(f + ahead, slot(f + ahead));
    }
    if (PROF && tid == 0) { const long long c = clock64(); tc += c - tck; tck = c; }
    const double* wlp;
    const double* wrp;
    if (plm) {
#pragma unroll
      for (int n = 0; n < 7; ++n) {
        const double q0 = P[slot(f)][n][tid];
        const double hdq = plm_half_slope(P[slot(f - 1)][n][tid], q0, P[slot(f + 1)][n][tid], ph.limiter);
        WL[f & 1][n][tid] = q0 + hdq;  // wL of face f+1
        WR[n][tid] = q0 - hdq;         // wR of face f
      }
      wlp = &WL[(f - 1) & 1][0][tid];
      wrp = &WR[0][tid];
    } else {
      wlp = &P[slot(f - 1)][0][tid];
      wrp = &P[slot(f)][0][tid];
    }
    if (PROF && tid == 0) { const long long c = clock64(); tp += c - tck; tck = c; }
    const int k = (DIR == 2) ? f : t, j = (DIR == 2) ? t : f;
    const int id = cid(f);
    PMHD_CHECK_ID(G, id);
    const double bn = __ldg(S[5 + DIR] + id);
    double out[8];
    int fb;
    if constexpr (PMHD_FLUX_SMEMW && (RS == PMHD_RIEMANN_HLLD || RS == PMHD_RIEMANN_ROE)) {
      const SmemW wl{wlp, MT}, wr{wrp, MT};
      fb = face_solve<RS>(wl, wr, bn, ph, c1024, out);
    } else {
      double wl[7], wr[7];
#pragma unroll
      for (int n = 0; n < 7; ++n) {
        wl[n] = wlp[n * MT];
        wr[n] = wrp[n * MT];
      }
      fb = face_solve<RS>(wl, wr, bn, ph, c1024, out);
    }
    if (fb) atomicAdd(&red[stage].fallback_count, 1ULL);
    double* const* F = B.fx[DIR];
    __stcs(F[0] + id, out[0]);
    __stcs(F[rot_var<DIR>(1)] + id, out[1]);
    __stcs(F[rot_var<DIR>(2)] + id, out[2]);
    __stcs(F[rot_var<DIR>(3)] + id, out[3]);
    __stcs(F[4] + id, out[4]);
    __stcs(F[5] + id, out[5]);
    __stcs(F[6] + id, out[6]);
    __stcs(F[7] + id, out[7]);
    if (reuse) rim_images<DIR>(blks, b, G, (G.dim == 3) ? 7 : 3, DIR, i, j, k, id, out);
    if (PROF && tid == 0) { const long long c = clock64(); tr += c - tck; tck = c; }
  }
  // donor cell with owned ranges: the cell-centred E row f_m1 is no face's
  // stencil cell here, but the update kernel's E box needs it
  if (write_ec && reuse && !plm && m1 == f_m1) cell(f_m1, slot(f_m1));
  if (PROF && tid == 0) {
    atomicAdd(&red[stage].phase[0], (unsigned long long)tc);
    atomicAdd(&red[stage].phase[1], (unsigned long long)tp);
    atomicAdd(&red[stage].phase[2], (unsigned long long)tr);
  }
}

//---------------------------------------------------------------------------
// Row-march flux kernel for the x1 faces.  Each warp owns one face row (j, k)
// and walks it in chunks of 32 faces: per chunk every lane loads and converts
// ONE cell (the one ahead of its face, so the last lane's slope has its right
// neighbour), the chunk's stencil is shared through a per-warp slice of
// shared memory (__syncwarp only: warps never wait for each other), each lane
// forms one PLM slope and solves one face; the two cells and the high-face
// state the next chunk needs from this one are carried in the slice, and the
// next chunk's raw values are loaded one chunk ahead into registers.  Same
// expressions and operand order as k_flux_fused: the same bits.
constexpr int XT = 128;  // 4 warps = 4 face rows
template <int RS, int MODE>
__global__ void __launch_bounds__(XT, MarchMinB<RS>::value)
k_flux_x1march(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, int sel, int plm, double c1024_arg,
               const KStage* __restrict__ kd, int stage, DevRed* red, int f_i0, int f_i1, int f_j0, int f_j1,
               int f_k0, int f_k1, int region, int reuse) {
  constexpr bool PROF = (MODE == 1);
  if (MODE == 2 && kd->skip) return;
  // per warp: Q[7][34] rotated primitives of cells fb-1 .. fb+32 (fb = the
  // chunk's first face), HI[7][33] high-face states of cells fb-1 .. fb+31,
  // LO[7][32] low-face states of cells fb .. fb+31
  __shared__ double Qs[4][7][34];
  __shared__ double HIs[4][7][33];
  __shared__ double LOs[4][7][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nj = f_j1 - f_j0, nrow = nj * (f_k1 - f_k0);
  const int b = blockIdx.y;
  const int row = blockIdx.x * 4 + warp;
  const DevBlock& B = blks[b];
  double* const* S = B.st[sel];
  if (region != 0) {  // as k_flux_fused, on the CTA's 4 rows (+ the i stencil)
    const int r0 = blockIdx.x * 4, r1 = min(r0 + 3, nrow - 1);
    const int ja = f_j0 + r0 % nj, ka = f_k0 + r0 / nj, jb = f_j0 + r1 % nj, kb = f_k0 + r1 / nj;
    const int jlo = (ka == kb) ? ja : f_j0, jhi = (ka == kb) ? jb : f_j1 - 1;
    bool inner = f_i0 - 2 >= G.is + 1 && f_i1 + 1 <= G.ie - 1 && jlo >= G.js + 1 && jhi <= G.je - 1;
    if (G.dim == 3) inner = inner && ka >= G.ks + 1 && kb <= G.ke - 1;
    if (inner != (region == 1)) return;
  }
  if (row >= nrow) return;  // (warp-uniform; no CTA barriers below)
  const int j = f_j0 + row % nj, k = f_k0 + row / nj;
  const bool rim = reuse && (f_i0 <= G.is || j <= G.js || j >= G.je - 1 ||
                             (G.dim == 3 && (k <= G.ks || k >= G.ke - 1)));
  double (*Q)[34] = Qs[warp];
  double (*HI)[33] = HIs[warp];
  double (*LO)[32] = LOs[warp];
  long long tc = 0, tp = 0, tr = 0, tck = 0;
  auto load_raw = [&](int i, double* ub) {
    if (i < 0 || i >= G.n1) return;
    const int id = G.idx(k, j, i);
    PMHD_CHECK_ID(G, id + G.sy);
#pragma unroll
    for (int v = 0; v < 5; ++v) ub[v] = __ldg(S[v] + id);
    ub[5] = __ldg(S[5] + id);
    ub[6] = __ldg(S[5] + id + 1);
    ub[7] = __ldg(S[6] + id);
    ub[8] = __ldg(S[6] + id + G.sx);
    ub[9] = __ldg(S[7] + id);
    ub[10] = __ldg(S[7] + id + G.sy);
  };
  // cons_to_prim of cell i from its raw values into Q[.][e]
  auto conv = [&](int i, int e, const double* ub) {
    if (i < 0 || i >= G.n1) return;
    double u[5], bc[3], w[8];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = ub[v];
    bc[0] = 0.5 * (ub[5] + ub[6]);
    bc[1] = 0.5 * (ub[7] + ub[8]);
    bc[2] = 0.5 * (ub[9] + ub[10]);
    const int fl = cons_to_prim(u, bc, ph, w, false);
    if ((fl & 4) && k >= G.ks && k < G.ke && j >= G.js && j < G.je && i >= G.is && i < G.ie) {
      const long long gi = (long long)B.c[0] * G.mb[0] + (i - G.is);
      const long long gj = (long long)B.c[1] * G.mb[1] + (j - G.js);
      const long long gk = (G.dim == 3) ? (long long)B.c[2] * G.mb[2] + (k - G.ks) : 0;
      atomicMin(&red[stage].bad_key, (unsigned long long)((gk * G.nx[1] + gj) * G.nx[0] + gi));
    }
#pragma unroll
    for (int n = 0; n < 7; ++n) Q[n][e] = w[rot_var<0>(n)];
  };
  const double c1024 = (MODE == 2) ? kd->c1024[0] : c1024_arg;
  if (PROF && lane == 0 && warp == 0) tck = clock64();
  // ---- prologue: cells fb-2 .. fb (lanes 0..2), then the high-face state of
  // cell fb-1 (PLM) -- what lane 0 of the first chunk takes from a previous one
  {
    double ub[11];
    const int i = f_i0 - 2 + lane;
    if (lane < 3) load_raw(i, ub);
    // (staged through Q[.][lane]: entries 0..2 = cells fb-2, fb-1, fb)
    if (lane < 3) conv(i, lane, ub);
    __syncwarp();
    double q0[7] = {}, q1[7] = {};
    if (lane == 0) {
#pragma unroll
      for (int n = 0; n < 7; ++n) {
        const double qm = Q[n][0], qc = Q[n][1], qp = Q[n][2];
        q0[n] = qc;
        q1[n] = qp;
        if (plm) HI[n][0] = qc + plm_half_slope(qm, qc, qp, ph.limiter);
      }
    }
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int n = 0; n < 7; ++n) {
        Q[n][0] = q0[n];  // cell fb-1
        Q[n][1] = q1[n];  // cell fb
      }
    }
  }
  double pre[11];
  load_raw(f_i0 + 1 + lane, pre);  // this lane's cell of the first chunk
  if (PROF && lane == 0 && warp == 0) { const long long c = clock64(); tc += c - tck; tck = c; }
  double* const* F = B.fx[0];
  for (int fb = f_i0; fb < f_i1; fb += 32) {
    // ---- cells fb+1 .. fb+32 (lane l: fb+1+l) into Q[.][2+l]; Q[.][0..1]
    // hold fb-1, fb (the previous chunk's last two cells)
    __syncwarp();
    conv(fb + 1 + lane, 2 + lane, pre);
    if (fb + 32 < f_i1) load_raw(fb + 33 + lane, pre);  // next chunk, one ahead
    __syncwarp();
    if (PROF && lane == 0 && warp == 0) { const long long c = clock64(); tc += c - tck; tck = c; }
    const int f = fb + lane;  // this lane's face: between cells f-1 (Q[.][lane]) and f (Q[.][lane+1])
    if (plm) {
#pragma unroll
      for (int n = 0; n < 7; ++n) {
        const double q0 = Q[n][lane + 1];
        const double hdq = plm_half_slope(Q[n][lane], q0, Q[n][lane + 2], ph.limiter);
        HI[n][lane + 1] = q0 + hdq;  // wL of face f+1
        LO[n][lane] = q0 - hdq;      // wR of face f
      }
      __syncwarp();
    }
    if (PROF && lane == 0 && warp == 0) { const long long c = clock64(); tp += c - tck; tck = c; }
    if (f < f_i1) {
      const int id = G.idx(k, j, f);
      PMHD_CHECK_ID(G, id);
      const double bn = __ldg(S[5] + id);
      double out[8];
      int fb2;
      if (plm) {
        const SmemW wl{&HI[0][lane], 33}, wr{&LO[0][lane], 32};
        fb2 = face_solve<RS>(wl, wr, bn, ph, c1024, out);
      } else {
        const SmemW wl{&Q[0][lane], 34}, wr{&Q[0][lane + 1], 34};
        fb2 = face_solve<RS>(wl, wr, bn, ph, c1024, out);
      }
      if (fb2) atomicAdd(&red[stage].fallback_count, 1ULL);
      __stcs(F[0] + id, out[0]);
      __stcs(F[1] + id, out[1]);
      __stcs(F[2] + id, out[2]);
      __stcs(F[3] + id, out[3]);
      __stcs(F[4] + id, out[4]);
      __stcs(F[5] + id, out[5]);
      __stcs(F[6] + id, out[6]);
      __stcs(F[7] + id, out[7]);
      if (rim) rim_images<0>(blks, b, G, (G.dim == 3) ? 7 : 3, 0, f, j, k, id, out);
    }
    if (PROF && lane == 0 && warp == 0) { const long long c = clock64(); tr += c - tck; tck = c; }
    // carry: cells fb+31, fb+32 -> Q[.][0..1]; high-face state of cell fb+31 -> HI[.][0]
    __syncwarp();
    if (lane < 2) {
#pragma unroll
      for (int n = 0; n < 7; ++n) Q[n][lane] = Q[n][32 + lane];
    }
    if (plm && lane == 2) {
#pragma unroll
      for (int n = 0; n < 7; ++n) HI[n][0] = HI[n][32];
    }
  }
  if (PROF && lane == 0 && warp == 0) {
    atomicAdd(&red[stage].phase[0], (unsigned long long)tc);
    atomicAdd(&red[stage].phase[1], (unsigned long long)tp);
    atomicAdd(&red[stage].phase[2], (unsigned long long)tr);
  }
}

//---------------------------------------------------------------------------
// x1 + x2 flux kernel (owned-face ranges only): one 32 x 16 tile of x1 AND
// x2 faces in one k-plane.  The flux kernels spend most of their time on
// loading, converting and reconstructing stencil cells and storing faces
// (with the Riemann solver replaced by a central flux a launch still takes
// 80 % of its time), so the two in-plane directions
// share one load + cons_to_prim of the union stencil (704 cells for 1024
// faces; separate x1 / x2 tiles convert 1184).  The PLM writes its interface
// values to a separate buffer (R) instead of in place, so a direction's
// reconstruction needs one barrier instead of one per variable.  Same
// expressions and operands as k_flux_fused: the same bits.
constexpr int XY_FX = 32, XY_FY = 16;          // faces per tile along i, j
constexpr int XY_NC = XY_FX + 4, XY_NR = XY_FY + 4;  // cell tile 36 x 20 (i0-2.., j0-2..)
constexpr int XY_NCELL = XY_NC * XY_NR;
constexpr int XY_R1 = (XY_FX + 1) * XY_FY;    // x1 reconstruction cells: i0-1..i0+31 x j0..j0+15
constexpr int XY_R2 = XY_FX * (XY_FY + 1);    // x2 reconstruction cells: i0..i0+31 x j0-1..j0+15
constexpr int XY_RS = XY_R2 > XY_R1 ? XY_R2 : XY_R1;
constexpr int XY_T = 256;
// side states in lab-order primitives, read in the rotated order of DIR
template <int DIR>
struct RotW {
  const volatile double* p;
  int s;
  PMHD_DEV double operator[](int n) const { return p[rot_var<DIR>(n) * s]; }
};

template <int RS, int MODE>
__global__ void __launch_bounds__(XY_T, 2)
k_flux_xy(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, int sel, int plm, double c1024x, double c1024y,
          const KStage* __restrict__ kd, int stage, DevRed* red, int write_ec) {
  constexpr bool PROF = (MODE == 1);
  if (MODE == 2 && kd->skip) return;
  extern __shared__ __align__(16) double xy_smem[];
  double* P = xy_smem;                  // [8][XY_NCELL] lab-order primitives
  double* R = xy_smem + 8 * XY_NCELL;   // [14][XY_RS]: 0..6 low-face (wR), 7..13 high-face (wL) values
  __shared__ long long tph[4];
  const int tid = threadIdx.x;
  if (PROF && tid == 0) tph[0] = clock64();
  const int nk = G.ke - G.ks;
  const int b = blockIdx.z / nk;
  const int k = G.ks + (int)(blockIdx.z % nk);
  const int fi0 = G.is + blockIdx.x * XY_FX, fj0 = G.js + blockIdx.y * XY_FY;
  const DevBlock& B = blks[b];
  double* const* S = B.st[sel];
  const bool rim = fi0 <= G.is || fi0 + XY_FX - 1 >= G.ie - 1 || fj0 <= G.js || fj0 + XY_FY - 1 >= G.je - 1 ||
                   (G.dim == 3 && (k <= G.ks || k >= G.ke - 1));
  // ---- phase 1: load + cons_to_prim of the union stencil ------------------
  // tile cell c = r * 36 + col <-> (i0 - 2 + col, j0 - 2 + r); PLM needs the
  // 16 main rows over all 36 columns and the 2 + 2 halo rows over the 32
  // face columns; donor cell the cells next to the faces only
  auto cell_ij = [&](int c, int& i, int& j) {
    const int col = c % XY_NC, row = c / XY_NC;
    i = fi0 - 2 + col;
    j = fj0 - 2 + row;
    const bool main_row = row >= 2 && row < XY_NR - 2;
    bool need;
    if (plm) need = main_row || (col >= 2 && col < XY_NC - 2);
    else {
      need = (main_row && col >= 1 && col < XY_NC - 2) || (row == 1 && col >= 2 && col < XY_NC - 2);
      // the cell-centred E row above the last face row (2D, last tile)
      if (write_ec && row == XY_NR - 2 && col >= 2 && col < XY_NC - 2 && fj0 + XY_FY == G.je) need = true;
    }
    return c < XY_NCELL && need && i >= 0 && i < G.n1 && j >= 0 && j < G.n2;
  };
  auto finish = [&](int c, int id, const double* ub) {
    double u[5], bc[3], w[8];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = ub[v];
    bc[0] = 0.5 * (ub[5] + ub[6]);
    bc[1] = 0.5 * (ub[7] + ub[8]);
    bc[2] = 0.5 * (ub[9] + ub[10]);
    const int fl = cons_to_prim(u, bc, ph, w, false);
    int i, j;
    cell_ij(c, i, j);
    if ((fl & 4) && k >= G.ks && k < G.ke && j >= G.js && j < G.je && i >= G.is && i < G.ie) {
      const long long gi = (long long)B.c[0] * G.mb[0] + (i - G.is);
      const long long gj = (long long)B.c[1] * G.mb[1] + (j - G.js);
      const long long gk = (G.dim == 3) ? (long long)B.c[2] * G.mb[2] + (k - G.ks) : 0;
      atomicMin(&red[stage].bad_key, (unsigned long long)((gk * G.nx[1] + gj) * G.nx[0] + gi));
    }
    if (write_ec) {  // 2D: this kernel is the last direction (rows js-1 .. je)
      const bool own = (j >= fj0 && j < fj0 + XY_FY) || (fj0 == G.js && j == G.js - 1) ||
                       (j == G.je && fj0 + XY_FY >= G.je);
      if (own && i >= G.is && i < G.ie) {
        const double ev[3] = {w[3] * w[6] - w[2] * w[7], w[1] * w[7] - w[3] * w[5], w[2] * w[5] - w[1] * w[6]};
        B.ec[0][id] = ev[0];
        B.ec[1][id] = ev[1];
        B.ec[2][id] = ev[2];
        if (rim) rim_images<3>(blks, b, G, 1, -1, i, j, k, id, ev);
      }
    }
#pragma unroll
    for (int v = 0; v < 8; ++v) P[v * XY_NCELL + c] = w[v];
  };
  constexpr int PER = (XY_NCELL + XY_T - 1) / XY_T;
  // all of this thread's cells' raw values in flight before any is converted
  double ub[PER][11];
  int cid[PER];
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int c = tid + p * XY_T;
    int i, j;
    cid[p] = -1;
    if (!cell_ij(c, i, j)) continue;
    const int id = G.idx(k, j, i);
    PMHD_CHECK_ID(G, id + G.sy);
    cid[p] = id;
#pragma unroll
    for (int v = 0; v < 5; ++v) ub[p][v] = __ldg(S[v] + id);
    ub[p][5] = __ldg(S[5] + id);
    ub[p][6] = __ldg(S[5] + id + 1);
    ub[p][7] = __ldg(S[6] + id);
    ub[p][8] = __ldg(S[6] + id + G.sx);
    ub[p][9] = __ldg(S[7] + id);
    ub[p][10] = __ldg(S[7] + id + G.sy);
  }
#pragma unroll
  for (int p = 0; p < PER; ++p)
    if (cid[p] >= 0) finish(tid + p * XY_T, cid[p], ub[p]);
  __syncthreads();
  if (PROF && tid == 0) tph[1] = clock64();
  long long trec = 0, trie = 0;

  // one direction: reconstruct (stage 2) then solve the tile's 512 faces
  auto direction = [&](auto dir_tag, double c1024) {
    constexpr int DIR = decltype(dir_tag)::value;
    constexpr int DC = (DIR == 0) ? 1 : XY_NC;     // stencil stride in the cell tile
    constexpr int NRC = (DIR == 0) ? XY_R1 : XY_R2;
    long long t0 = 0;
    if (PROF && tid == 0) t0 = clock64();
    if (plm) {
      for (int q = tid; q < NRC; q += XY_T) {
        // reconstruction cell q -> tile cell
        const int c = (DIR == 0) ? (q / (XY_FX + 1) + 2) * XY_NC + (q % (XY_FX + 1)) + 1
                                 : (q / XY_FX + 1) * XY_NC + (q % XY_FX) + 2;
#pragma unroll
        for (int n = 0; n < 7; ++n) {
          const double* pv = P + rot_var<DIR>(n) * XY_NCELL + c;
          const double q0 = pv[0];
          const double hdq = plm_half_slope(pv[-DC], q0, pv[DC], ph.limiter);
          R[n * XY_RS + q] = q0 - hdq;        // wR of the face below
          R[(7 + n) * XY_RS + q] = q0 + hdq;  // wL of the face above
        }
      }
      __syncthreads();
    }
    if (PROF && tid == 0) { const long long t = clock64(); trec += t - t0; t0 = t; }
    double* const* F = B.fx[DIR];
    for (int h = 0; h < 2; ++h) {
      const int fq = tid + XY_T * h;  // face in the tile: 32 along i, 16 along j
      const int fc = fq % XY_FX, fr = fq / XY_FX;
      const int i = fi0 + fc, j = fj0 + fr;
      if (i >= G.ie || j >= G.je) continue;
      const int id = G.idx(k, j, i);
      PMHD_CHECK_ID(G, id);
      const double bn = __ldg(S[5 + DIR] + id);
      double out[8];
      int fb;
      if (plm) {
        // reconstruction cells of the face's low / high sides
        const int ql = (DIR == 0) ? fr * (XY_FX + 1) + fc : fr * XY_FX + fc;
        const int qh = (DIR == 0) ? ql + 1 : ql + XY_FX;
        const SmemW wl{R + 7 * XY_RS + ql, XY_RS}, wr{R + qh, XY_RS};
        fb = face_solve<RS>(wl, wr, bn, ph, c1024, out);
      } else {
        const int ch = (fr + 2) * XY_NC + fc + 2, cl = ch - DC;
        const RotW<DIR> wl{P + cl, XY_NCELL}, wr{P + ch, XY_NCELL};
        fb = face_solve<RS>(wl, wr, bn, ph, c1024, out);
      }
      if (fb) atomicAdd(&red[stage].fallback_count, 1ULL);
      __stcs(F[0] + id, out[0]);
      __stcs(F[rot_var<DIR>(1)] + id, out[1]);
      __stcs(F[rot_var<DIR>(2)] + id, out[2]);
      __stcs(F[rot_var<DIR>(3)] + id, out[3]);
      __stcs(F[4] + id, out[4]);
      __stcs(F[5] + id, out[5]);
      __stcs(F[6] + id, out[6]);
      __stcs(F[7] + id, out[7]);
      if (rim) rim_images<DIR>(blks, b, G, (G.dim == 3) ? 7 : 3, DIR, i, j, k, id, out);
    }
    if (PROF && tid == 0) trie += clock64() - t0;
  };
  direction(std::integral_constant<int, 0>{}, (MODE == 2) ? kd->c1024[0] : c1024x);
  if (plm) __syncthreads();  // R is refilled by x2
  direction(std::integral_constant<int, 1>{}, (MODE == 2) ? kd->c1024[1] : c1024y);
  if (PROF && tid == 0) {
    atomicAdd(&red[stage].phase[0], (unsigned long long)(tph[1] - tph[0]));
    atomicAdd(&red[stage].phase[1], (unsigned long long)trec);
    atomicAdd(&red[stage].phase[2], (unsigned long long)trie);
  }
}

}  // namespace

// slab / nslab / S: k-slab pipelining (pmhd_gpu.cu): slab q covers k planes
// [ks + q S, ks + (q+1) S) of x1/x2 faces (the first slab also ks-1, the last
// up to ke) and x3 face planes [ks + q S, ...) (the last up to ke); S is a
// multiple of the x3 tile's FS (16).  nslab = 1 is the whole block.
void launch_flux_fused(const DevBlock* blks, const KGeom& G, const KPhys& ph, int dir, int sel,
                       int plm, double c1024, const KStage* kd, int stage, DevRed* red, int slab,
                       int nslab, int S, cudaStream_t s, int region, const FluxOpts& opt) {
  const int reuse = opt.reuse;
  const int d3 = (G.dim == 3) ? 1 : 0;
  // face ranges of the oracle: [lo, hi) per axis;
  // with owned-face reuse [s, e) on every axis (the rest are rim images)
  int i0, i1, j0, j1, k0, k1;
  if (reuse) { k0 = G.ks; k1 = G.ke; j0 = G.js; j1 = G.je; i0 = G.is; i1 = G.ie; }
  else if (dir == 0) { k0 = G.ks - d3; k1 = G.ke + d3; j0 = G.js - 1; j1 = G.je + 1; i0 = G.is; i1 = G.ie + 1; }
  else if (dir == 1) { k0 = G.ks - d3; k1 = G.ke + d3; j0 = G.js; j1 = G.je + 1; i0 = G.is - 1; i1 = G.ie + 1; }
  else { k0 = G.ks; k1 = G.ke + 1; j0 = G.js - 1; j1 = G.je + 1; i0 = G.is - 1; i1 = G.ie + 1; }
  const int ns0 = (dir == 2) ? k0 : j0, ns1 = (dir == 2) ? k1 : j1;
  int nt0 = (dir == 2) ? j0 : k0, nt1 = (dir == 2) ? j1 : k1;
  const int write_ec = (dir == G.dim - 1) ? 1 : 0;
  const int FX = (dir == 0) ? TileShape<0>::FX : TileShape<1>::FX;
  const int FS = (dir == 0) ? TileShape<0>::FS : TileShape<1>::FS;
  int ty0 = 0, ty1 = (ns1 - ns0 + FS - 1) / FS;
  if (nslab > 1) {
    const bool first = (slab == 0), last = (slab == nslab - 1);
    if (dir == 2) {  // k is the tile's second axis (face planes)
      ty0 = slab * S / FS;
      if (!last) ty1 = (slab + 1) * S / FS;
    } else {         // k is the launch's third axis
      const int a = first ? nt0 : G.ks + slab * S;
      const int e = last ? nt1 : G.ks + (slab + 1) * S;
      nt0 = a;
      nt1 = e;
    }
  }
  // x2 / x3 faces: the column-march kernel (PMHD_FLUX_MARCH=0: the tile
  // kernel).  Measured at 256^3 per cycle: 7.56 ms against 7.73 for the tile
  // kernel with the next cell's raw values prefetched one step ahead; 7.80
  // without the prefetch (4 CTAs/SM), 7.93 at 5 CTAs/SM (spills)
  // (PMHD_FLUX_MARCH=2 forces the march on any mesh size)
  const int march_mode = opt.march;
  const bool march_on = march_mode != 0 && ((opt.march_stages >> (plm ? 1 : 0)) & 1);
  // x1 faces: the row-march kernel (stage 2 by default; PMHD_FLUX_MARCH_X1=0:
  // the x1 tile kernel).  Measured at 256^3 per cycle with the marches in
  // stage 2 only: 7.45-7.47 ms with the x1 row march, 7.53 without; in both
  // stages 7.57-7.60 either way
  const int nrow = (j1 - j0) * (k1 - k0);
  const dim3 xg((nrow + 3) / 4, G.nb, 1);
  const bool x1_fills = march_mode == 2 || (long long)xg.x * xg.y >= 2LL * 148 * PMHD_MARCH_MINB;
  if (dir == 0 && march_on && opt.march_x1 && x1_fills && nslab == 1) {
#define PMHD_X1M_LAUNCH(R, M) \
  k_flux_x1march<R, M><<<xg, XT, 0, s>>>(blks, G, ph, sel, plm, c1024, kd, stage, red, i0, i1, j0, j1, k0, k1, \
                                         region, reuse)
#define PMHD_X1M_MODES(R)                              \
  do {                                                 \
    if (kd) PMHD_X1M_LAUNCH(R, 2);                     \
    else if (ph.prof) PMHD_X1M_LAUNCH(R, 1);           \
    else PMHD_X1M_LAUNCH(R, 0);                        \
  } while (0)
    if (ph.riemann == PMHD_RIEMANN_HLLE) PMHD_X1M_MODES(PMHD_RIEMANN_HLLE);
    else if (ph.riemann == PMHD_RIEMANN_ROE) PMHD_X1M_MODES(PMHD_RIEMANN_ROE);
    else PMHD_X1M_MODES(PMHD_RIEMANN_HLLD);
#undef PMHD_X1M_MODES
#undef PMHD_X1M_LAUNCH
    return;
  }
  // march axis m: j for x2, k for x3; transverse t: k for x2, j for x3
  const int mm0 = (dir == 2) ? k0 : j0, mm1 = (dir == 2) ? k1 : j1;
  const int mt0 = (dir == 2) ? j0 : k0, mt1 = (dir == 2) ? j1 : k1;
  const dim3 mg((i1 - i0 + 31) / 32, (mt1 - mt0 + 3) / 4, ((mm1 - mm0 + PMHD_MARCH_L - 1) / PMHD_MARCH_L) * G.nb);
  // one thread per face column: small meshes (a 64^3 block: 96 CTAs; the
  // 512^2 Orszag-Tang in 128^2 blocks: 384) cannot fill the GPU that way,
  // so below two full waves of 148 SMs the tile kernel runs instead
  const bool march_fills = march_mode == 2 || (long long)mg.x * mg.y * mg.z >= 2LL * 148 * PMHD_MARCH_MINB;
  if (dir >= 1 && march_on && march_fills && nslab == 1) {
    const int m0 = mm0, m1 = mm1, t0 = mt0, t1 = mt1;
#define PMHD_MARCH_LAUNCH(D, R, M) \
  k_flux_march<D, R, M><<<mg, MT, 0, s>>>(blks, G, ph, sel, plm, c1024, kd, stage, red, write_ec, i0, i1, m0, m1, \
                                          t0, t1, region, reuse)
#define PMHD_MARCH_MODES(D, R)                                     \
  do {                                                             \
    if (kd) PMHD_MARCH_LAUNCH(D, R, 2);                            \
    else if (ph.prof) PMHD_MARCH_LAUNCH(D, R, 1);                  \
    else PMHD_MARCH_LAUNCH(D, R, 0);                               \
  } while (0)
#define PMHD_MARCH_DIRS(R)                                         \
  do {                                                             \
    if (dir == 1) PMHD_MARCH_MODES(1, R);                          \
    else PMHD_MARCH_MODES(2, R);                                   \
  } while (0)
    if (ph.riemann == PMHD_RIEMANN_HLLE) PMHD_MARCH_DIRS(PMHD_RIEMANN_HLLE);
    else if (ph.riemann == PMHD_RIEMANN_ROE) PMHD_MARCH_DIRS(PMHD_RIEMANN_ROE);
    else PMHD_MARCH_DIRS(PMHD_RIEMANN_HLLD);
#undef PMHD_MARCH_DIRS
#undef PMHD_MARCH_MODES
#undef PMHD_MARCH_LAUNCH
    return;
  }
  const dim3 grid((i1 - i0 + FX - 1) / FX, ty1 - ty0, (nt1 - nt0) * G.nb);
  // experiment knob (PMHD_FLUX_SMEM_PAD = bytes of unused dynamic shared
  // memory per CTA): caps the flux CTAs per SM so that an update CTA of a
  // concurrent stream can co-reside (k-slab pipeline study)
  const int pad = opt.pad ? opt.pad + (dir == 0 ? 1792 : 0) : 0;
#define PMHD_FLUX_LAUNCH(D, R)                                                                      \
  do {                                                                                              \
    if (kd)                                                                                         \
      k_flux_fused<D, R, 2><<<grid, NTHR, pad, s>>>(blks, G, ph, sel, plm, c1024, kd, stage, red,     \
                                                  write_ec, i0, i1, ns0, ns1, nt0, nt1, ty0, region, reuse); \
    else if (ph.prof)                                                                               \
      k_flux_fused<D, R, 1><<<grid, NTHR, pad, s>>>(blks, G, ph, sel, plm, c1024, kd, stage, red,     \
                                                  write_ec, i0, i1, ns0, ns1, nt0, nt1, ty0, region, reuse); \
    else                                                                                            \
      k_flux_fused<D, R, 0><<<grid, NTHR, pad, s>>>(blks, G, ph, sel, plm, c1024, kd, stage, red,     \
                                                  write_ec, i0, i1, ns0, ns1, nt0, nt1, ty0, region, reuse); \
  } while (0)
#define PMHD_FLUX_DIRS(R)                          \
  do {                                             \
    if (dir == 0) PMHD_FLUX_LAUNCH(0, R);          \
    else if (dir == 1) PMHD_FLUX_LAUNCH(1, R);     \
    else PMHD_FLUX_LAUNCH(2, R);                   \
  } while (0)
  if (ph.riemann == PMHD_RIEMANN_HLLE) PMHD_FLUX_DIRS(PMHD_RIEMANN_HLLE);
  else if (ph.riemann == PMHD_RIEMANN_ROE) PMHD_FLUX_DIRS(PMHD_RIEMANN_ROE);
  else PMHD_FLUX_DIRS(PMHD_RIEMANN_HLLD);
#undef PMHD_FLUX_DIRS
#undef PMHD_FLUX_LAUNCH
}

// x1 + x2 faces in one launch (owned-face ranges only; see k_flux_xy)
void launch_flux_xy(const DevBlock* blks, const KGeom& G, const KPhys& ph, int sel, int plm, double c1024x,
                    double c1024y, const KStage* kd, int stage, DevRed* red, cudaStream_t s) {
  const int write_ec = (G.dim == 2) ? 1 : 0;
  const dim3 grid((G.ie - G.is + XY_FX - 1) / XY_FX, (G.je - G.js + XY_FY - 1) / XY_FY, (G.ke - G.ks) * G.nb);
  constexpr int smem_max = (8 * XY_NCELL + 14 * XY_RS) * 8;
  const int smem = plm ? smem_max : 8 * XY_NCELL * 8;  // donor cell: no reconstruction buffer
#define PMHD_XY_LAUNCH(R)                                                                               \
  do {                                                                                                  \
    static std::atomic<unsigned long long> attr_devs{0};                                                \
    int dev = 0;                                                                                        \
    cudaGetDevice(&dev);                                                                                \
    if (!(attr_devs.load() & (1ULL << (dev & 63)))) {                                                   \
      cudaFuncSetAttribute(k_flux_xy<R, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);     \
      cudaFuncSetAttribute(k_flux_xy<R, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);     \
      cudaFuncSetAttribute(k_flux_xy<R, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);     \
      attr_devs.fetch_or(1ULL << (dev & 63));                                                           \
    }                                                                                                   \
    if (kd) k_flux_xy<R, 2><<<grid, XY_T, smem, s>>>(blks, G, ph, sel, plm, c1024x, c1024y, kd, stage, red, write_ec); \
    else if (ph.prof) k_flux_xy<R, 1><<<grid, XY_T, smem, s>>>(blks, G, ph, sel, plm, c1024x, c1024y, kd, stage, red, write_ec); \
    else k_flux_xy<R, 0><<<grid, XY_T, smem, s>>>(blks, G, ph, sel, plm, c1024x, c1024y, kd, stage, red, write_ec); \
  } while (0)
  if (ph.riemann == PMHD_RIEMANN_HLLE) PMHD_XY_LAUNCH(PMHD_RIEMANN_HLLE);
  else if (ph.riemann == PMHD_RIEMANN_ROE) PMHD_XY_LAUNCH(PMHD_RIEMANN_ROE);
  else PMHD_XY_LAUNCH(PMHD_RIEMANN_HLLD);
#undef PMHD_XY_LAUNCH
}

}  // namespace pmhd_gpu
