// kernels_update_tma.cu -- the fused end of a VL2 stage for 3D meshes with
// its operands staged in shared memory by TMA (cp.async.bulk.tensor).
//
// Same reference ops, same expressions and operand order as k_update_fused
// (kernels_update.cu), so results are bit-identical to it and to the oracle:
// corner EMFs (ct_emf), constrained-transport face update
// (ct_update_face_b), conserved update ("integrate",
// SPEC.md:212, :527), face_to_center_b + end-of-stage cons_to_prim with
// floors / error detection and the compute_dt
// partial min.
//
// Why a second kernel.  k_update_fused is latency-bound (ncu: 4.3 TB/s, 52 %
// DRAM throughput, long-scoreboard stalls): every phase of its k-march loads
// its operands with LDG into a 48-register budget, so only a few loads per
// thread are in flight between the phase barriers.  Here one thread issues
// the whole next plane's operands as TMA boxes into a two-slot ring while the
// CTA computes the current plane from shared memory:
//   EMF group  (per plane p; box 34 x 10 cells from (i0-1, j0-1)): the face E
//              and upwind weights X1/X2[5..7] at plane p, X3[5..7] at x3 face
//              p, the cell-centred E of plane p -- 12 boxes, 32.6 KB;
//   cell group (per plane p; boxes of 32-34 x 8-9 from (i0, j0)): the hydro
//              fluxes X1/X2[0..4] at plane p and X3[0..4] at face p+1, the
//              base state u^n (5 conserved + 3 face-B; b3 at face p+1) --
//              22 boxes, 46.7 KB.
// A step k (cells of plane k) computes E3(k) and E1/E2(k+1/2) from EMF slots
// k and k+1, then refills slot k with plane k+2; the cell group of plane k+1
// is issued at the start of step k.  The x3 fluxes at face k are carried in
// registers from the previous step.  Tiles of 32 x 4 cells (PMHD_UPDATE_TMA_TY)
// with two threads per cell and ~106 KB of shared memory: two CTAs per SM.
// The EMF, CT and dt work is spread over all threads as flat, balanced item
// lists, the conserved update and cons_to_prim over the first half.
// (Measured at 256^3: a 32 x 8 tile with one CTA of 256 threads per SM ran
// at 8 warps, IPC 0.93, 1.93 ms per launch; with 512 threads 1.69 ms; the
// LDG kernel takes 1.56 ms -- with one CTA per SM every barrier drains the
// SM.)
#include <atomic>

#include "kernels.cuh"
#include "tma.cuh"

namespace pmhd_gpu {

namespace {

#ifndef PMHD_UPDATE_TMA_TY
#define PMHD_UPDATE_TMA_TY 4  // tile rows: 4 -> two CTAs per SM (8: one CTA of 512 threads)
#endif
constexpr int TX = 32, TY = PMHD_UPDATE_TMA_TY, NC = TX * TY;  // NC cells per tile
constexpr int NT = 2 * NC;                                       // threads (2 per cell)
constexpr int MINB = (TY == 8) ? 1 : 2;                          // CTAs per SM
__host__ __device__ constexpr int pad16(int n) { return (n + 15) / 16 * 16; }  // 128 B multiple
// A TMA box must start on a 16-byte boundary in global memory (a box whose
// first element is 8 B off faults with "illegal instruction").  With the
// ABI's row alignment (face-data rows aligned at i = is, state and cell-E
// rows at i = is-1) and even tile origins i0 - is, face-data boxes start at
// even offsets from i0 and state / cell-E boxes at odd ones; the host checks
// this per map (build_update_maps) and keeps the LDG kernel otherwise.
// EMF group: cells i0-1 .. i0+32, rows j0-1 .. j0+TY -- face data from i0-2
// (36 wide), cell E from i0-1 (34 wide).
constexpr int EBH = TY + 2, EBOX = pad16(36 * EBH);
constexpr int NEMF = 12;              // EMF-group arrays (ids 0..11)
__host__ __device__ constexpr int ew(int a) { return a < 9 ? 36 : 34; }  // EMF box width
__host__ __device__ constexpr int eo(int a) { return a < 9 ? 1 : 0; }    // column of cell i0-1
// cell-group boxes (doubles) and their offsets in a slot (all 128 B multiples)
constexpr int BX1 = 34 * TY;          // X1[0..4] at plane p, [TY][34] from i0
constexpr int BX2 = 32 * (TY + 1);    // X2[0..4] at plane p, [TY+1][32] from i0
constexpr int BSB = 34 * TY;          // u^n[0..4], b1f^n at plane p, b3f^n at face p+1: [TY][34] from i0-1
constexpr int BS6 = 34 * (TY + 1);    // b2f^n at plane p, [TY+1][34] from i0-1
constexpr int BC = 32 * TY;           // X3[0..4] at face p+1, [TY][32] from i0
constexpr int OX1 = 0;
constexpr int OX2 = OX1 + 5 * pad16(BX1);
constexpr int OSB = OX2 + 5 * pad16(BX2);
constexpr int OS5 = OSB + 5 * pad16(BSB);
constexpr int OS6 = OS5 + pad16(BSB);
constexpr int OX3 = OS6 + pad16(BS6);
constexpr int OS7 = OX3 + 5 * pad16(BC);
constexpr int CSLOT = OS7 + pad16(BSB);  // doubles per cell slot
constexpr int SX1 = pad16(BX1), SX2 = pad16(BX2), SSB = pad16(BSB), SC = pad16(BC);  // box strides
constexpr unsigned EMF_BYTES = (9 * 36 + 3 * 34) * EBH * 8u;
constexpr unsigned CELL_BYTES = (5 * BX1 + 5 * BX2 + 5 * BSB + BSB + BS6 + 5 * BC + BSB) * 8u;

// Map ids per block (kMaps per block and table parity; see build_update_maps)
//  0..2  X1[5..7]   3..5  X2[5..7]   6..8  X3[5..7]   9..11 E_cell[0..2]
// 12..16 X1[0..4]  17..21 X2[0..4]  22..26 X3[0..4]  27..31 u^n[0..4]
// 32 b1f^n  33 b2f^n  34 b3f^n
constexpr int kMaps = 35;
// first cell of map id a's box relative to the tile origin i0
__host__ __device__ constexpr int box_i(int a) { return a < 9 ? -2 : (a < 12 ? -1 : (a < 27 ? 0 : -1)); }

#ifndef PMHD_UPDATE_STCS
#define PMHD_UPDATE_STCS 1
#endif
__device__ __forceinline__ void ST(double* p, double v) {
#if PMHD_UPDATE_STCS
  __stcs(p, v);
#else
  *p = v;
#endif
}

struct alignas(128) TSmem {
  double emf[2][NEMF][EBOX];
  double cell[2][CSLOT];
  double e3s[TY + 1][TX + 1];   // E3 at (k, j-1/2, i-1/2)
  double e1s[2][TY + 1][TX];    // E1 at (k -/+ 1/2, j-1/2, i), slot by parity
  double e2s[2][TY][TX + 1];    // E2 at (k -/+ 1/2, j, i-1/2)
  double b1s[TY][TX + 1];
  double b2s[TY + 1][TX];
  double b3s[2][TY][TX];        // new b3 at faces k / k+1, slot by parity
  double wv[8][NC];             // end-of-stage primitives (dt terms)
  double redbuf[NT / 32];
  unsigned long long ebar[2], cbar[2];
  long long tph[3];
};
// (228 KB of shared memory per SM, 1 KB of it reserved per resident CTA)
static_assert(sizeof(TSmem) + 128 + 1024 <= 233472 / MINB, "shared memory budget (MINB CTAs per SM)");

// MODE: 0 product, 1 region profiling, 2 graph-replayed cycle (stage from kd)
template <int SEG, int MODE>
__global__ void __launch_bounds__(NT, MINB)
k_update_tma(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, KStage ks_arg, const KStage* __restrict__ kd,
             DevRed* red, int want_dt, int kr0, int kr1, const CUtensorMap* __restrict__ maps,
             unsigned long long xoffm, int push) {
  constexpr bool PROF = (MODE == 1);
  if (MODE == 2 && kd->skip) return;  // replayed cycle past the end of the run
  const KStage ks = (MODE == 2) ? *kd : ks_arg;
  extern __shared__ __align__(16) unsigned char upd_tma_smem[];
  TSmem& SM = *reinterpret_cast<TSmem*>((reinterpret_cast<uintptr_t>(upd_tma_smem) + 127) & ~uintptr_t(127));

  const int nseg = (kr1 - kr0 + SEG - 1) / SEG;
  const int b = blockIdx.z / nseg;
  const int kb = kr0 + (int)(blockIdx.z % nseg) * SEG;
  const int kend = min(kb + SEG, kr1);
  const int i0 = G.is + blockIdx.x * TX, j0 = G.js + blockIdx.y * TY;
  const int nx = min(TX, G.ie - i0), ny = min(TY, G.je - j0);
  const DevBlock& B = blks[b];
  const CUtensorMap* M = maps + kMaps * b;
  double* const* Sout = B.st[ks.out_sel];
  const int sy = G.sy;
  const int tid = threadIdx.x, tx = tid % TX, ty = (tid / TX) % TY;  // cell of threads < NC
  const int mode = ph.emf;
  const double c1 = ks.c1, c2 = ks.c2, c3 = ks.c3;
  if (PROF && tid == 0) { SM.tph[0] = clock64(); SM.tph[1] = SM.tph[2] = 0; }
  // x1 ghost push (see k_update_fused): the left / right neighbour's arrays
  double* const* PL = push ? blks[B.nbr[0][0]].st[ks.out_sel] : nullptr;
  double* const* PR = push ? blks[B.nbr[0][1]].st[ks.out_sel] : nullptr;
  auto push_cell = [&](int v, int i, int id, double val) {
    if (i < G.is + G.ng) { PMHD_CHECK_ID(G, id + G.mb[0]); ST(PL[v] + id + G.mb[0], val); }
    if (i >= G.ie - G.ng) { PMHD_CHECK_ID(G, id - G.mb[0]); ST(PR[v] + id - G.mb[0], val); }
  };

  // ---- TMA issue (thread 0) ---------------------------------------------------
  auto xo = [&](int a) { return (int)((xoffm >> a) & 1ull); };
  auto issue_emf = [&](int p) {  // EMF group of plane p into slot p & 1
#if defined(PMHD_TMA_DBG) && (PMHD_TMA_DBG == 1 || PMHD_TMA_DBG == 3)
    return;
#endif
    const int sl = p & 1;
    fence_proxy_async_smem();
    mbar_expect_tx(&SM.ebar[sl], EMF_BYTES);
#pragma unroll 1
    for (int a = 0; a < NEMF; ++a)
      tma_load_3d(&SM.emf[sl][a][0], M + a, &SM.ebar[sl], i0 + box_i(a) + xo(a), j0 - 1, p);
  };
  auto issue_cell = [&](int p) {  // cell group of plane p into slot p & 1
#if defined(PMHD_TMA_DBG) && (PMHD_TMA_DBG == 1 || PMHD_TMA_DBG == 2)
    return;
#endif
    const int sl = p & 1;
    double* C = SM.cell[sl];
    fence_proxy_async_smem();
    mbar_expect_tx(&SM.cbar[sl], CELL_BYTES);
#pragma unroll 1
    for (int v = 0; v < 5; ++v) {
      tma_load_3d(C + OX1 + v * SX1, M + 12 + v, &SM.cbar[sl], i0 + xo(12 + v), j0, p);
      tma_load_3d(C + OX2 + v * SX2, M + 17 + v, &SM.cbar[sl], i0 + xo(17 + v), j0, p);
      tma_load_3d(C + OSB + v * SSB, M + 27 + v, &SM.cbar[sl], i0 - 1 + xo(27 + v), j0, p);
      tma_load_3d(C + OX3 + v * SC, M + 22 + v, &SM.cbar[sl], i0 + xo(22 + v), j0, p + 1);
    }
    tma_load_3d(C + OS5, M + 32, &SM.cbar[sl], i0 - 1 + xo(32), j0, p);
    tma_load_3d(C + OS6, M + 33, &SM.cbar[sl], i0 - 1 + xo(33), j0, p);
    tma_load_3d(C + OS7, M + 34, &SM.cbar[sl], i0 - 1 + xo(34), j0, p + 1);
  };
  unsigned eph = 0u, cph = 0u;  // barrier phase bit of each ring slot (bit = slot)
  auto wait_emf = [&](int p) {
#if defined(PMHD_TMA_DBG) && (PMHD_TMA_DBG == 1 || PMHD_TMA_DBG == 3)
    return;
#endif
    const int sl = p & 1;
    mbar_wait(&SM.ebar[sl], (eph >> sl) & 1u);
    eph ^= 1u << sl;
  };
  auto wait_cell = [&](int p) {
#if defined(PMHD_TMA_DBG) && (PMHD_TMA_DBG == 1 || PMHD_TMA_DBG == 2)
    return;
#endif
    const int sl = p & 1;
    mbar_wait(&SM.cbar[sl], (cph >> sl) & 1u);
    cph ^= 1u << sl;
  };
  // EMF box element of array a at box row r (j0-1+r), column c (i0-1+c)
  auto E = [&](int sl, int a, int r, int c) -> double { return SM.emf[sl][a][r * ew(a) + c + eo(a)]; };

  // EMF items, one flat list so the 512 threads share them evenly: E3 at
  // plane k from slot e3 ([0, 297)), then E1 ([297, 585)) and E2 ([585, 849))
  // on the edge plane between planes (slot pm) and (slot pa), i.e. at kk - 1/2
  // for pa = slot of kk, into e1s / e2s[h]; same operands as k_update_fused
  // (X3 of face kk lives in the EMF slot of plane kk)
  constexpr int NE3 = (TY + 1) * (TX + 1), NE1 = (TY + 1) * TX, NE2 = TY * (TX + 1);
  auto emf_items = [&](int q0, int e3, int pa, int pm, int h) {
    for (int q = q0 + tid; q < NE3 + NE1 + NE2; q += NT) {
      if (q < NE3) {
        const int c = q % (TX + 1), r = q / (TX + 1);
        if (c > nx || r > ny) continue;
        SM.e3s[r][c] = corner_emf(mode, E(e3, 0, r + 1, c + 1), E(e3, 0, r, c + 1), E(e3, 4, r + 1, c + 1),
                                  E(e3, 4, r + 1, c), E(e3, 2, r + 1, c + 1), E(e3, 2, r, c + 1),
                                  E(e3, 5, r + 1, c + 1), E(e3, 5, r + 1, c), E(e3, 11, r + 1, c + 1),
                                  E(e3, 11, r + 1, c), E(e3, 11, r, c + 1), E(e3, 11, r, c));
      } else if (q < NE3 + NE1) {
        const int q1 = q - NE3, c = q1 % TX, r = q1 / TX;
        if (c >= nx || r > ny) continue;
        SM.e1s[h][r][c] = corner_emf(mode, E(pa, 3, r + 1, c + 1), E(pm, 3, r + 1, c + 1), E(pa, 7, r + 1, c + 1),
                                     E(pa, 7, r, c + 1), E(pa, 5, r + 1, c + 1), E(pm, 5, r + 1, c + 1),
                                     E(pa, 8, r + 1, c + 1), E(pa, 8, r, c + 1), E(pa, 9, r + 1, c + 1),
                                     E(pa, 9, r, c + 1), E(pm, 9, r + 1, c + 1), E(pm, 9, r, c + 1));
      } else {
        const int q2 = q - NE3 - NE1, c = q2 % (TX + 1), r = q2 / (TX + 1);
        if (c > nx || r >= ny) continue;
        SM.e2s[h][r][c] = corner_emf(mode, E(pa, 6, r + 1, c + 1), E(pa, 6, r + 1, c), E(pa, 1, r + 1, c + 1),
                                     E(pm, 1, r + 1, c + 1), E(pa, 8, r + 1, c + 1), E(pa, 8, r + 1, c),
                                     E(pa, 2, r + 1, c + 1), E(pm, 2, r + 1, c + 1), E(pa, 10, r + 1, c + 1),
                                     E(pm, 10, r + 1, c + 1), E(pa, 10, r + 1, c), E(pm, 10, r + 1, c));
      }
    }
  };

  // ---- prologue: EMF planes kb-1, kb and the cell group of kb in flight ------
  if (tid == 0) {
    mbar_init(&SM.ebar[0], 1);
    mbar_init(&SM.ebar[1], 1);
    mbar_init(&SM.cbar[0], 1);
    mbar_init(&SM.cbar[1], 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0) {
    issue_emf(kb - 1);
    issue_emf(kb);
    issue_cell(kb);
  }
  const bool own = (tid < NC) && (tx < nx) && (ty < ny);
  // the x3 fluxes at the lower face of this thread's cell (carried from one
  // step to the next afterwards) and b3f^n at face kb
  double x3lo[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  double b3lo = 0.0;
  if (own) {
    const int id = G.idx(kb, j0 + ty, i0 + tx);
    PMHD_CHECK_ID(G, id);
#pragma unroll
    for (int v = 0; v < 5; ++v) x3lo[v] = __ldg(B.fx[2][v] + id);
    b3lo = __ldg(B.st[0][7] + id);
  }
  wait_emf(kb - 1);
  wait_emf(kb);
  emf_items(NE3, 0, kb & 1, (kb - 1) & 1, kb & 1);  // E1 / E2 at kb - 1/2 (no E3)
  __syncthreads();
  if (tid == 0 && kb + 1 <= kend) issue_emf(kb + 1);  // into the slot of kb - 1, read just above
  if (own) {  // new b3 at face kb (face_b3 of k_update_fused)
    const int h = kb & 1;
    SM.b3s[h][ty][tx] = b3lo - (c1 * (SM.e2s[h][ty][tx + 1] - SM.e2s[h][ty][tx]) -
                                c2 * (SM.e1s[h][ty + 1][tx] - SM.e1s[h][ty][tx]));
  }

  double tmin = 1.0e300;
  for (int k = kb; k < kend; ++k) {
    const int lo = k & 1, hi = lo ^ 1;  // slots of planes k / k+1, edges k -/+ 1/2
    if (PROF && tid == 0 && k > kb) { const long long t = clock64(); SM.tph[2] += t - SM.tph[0]; SM.tph[0] = t; }
    // the next plane's cell group: its slot was last read in step k-1
    if (tid == 0 && k + 1 < kend) issue_cell(k + 1);
    wait_emf(k + 1);
    // ---- E3 at plane k, E1 / E2 at k + 1/2 ------------------------------------
    emf_items(0, lo, hi, lo, hi);
    __syncthreads();
    if (tid == 0 && k + 2 <= kend) issue_emf(k + 2);  // into slot lo: plane k was last read just above
    if (PROF && tid == 0) { const long long t = clock64(); SM.tph[1] += t - SM.tph[0]; SM.tph[0] = t; }
    wait_cell(k);
    const double* C = SM.cell[lo];
    // ---- constrained-transport face update: b1f (faces i0 .. i0+nx), b2f
    // (faces j0 .. j0+ny), b3f at face k+1 (face k carried); one flat list
    constexpr int NB1 = TY * (TX + 1), NB2 = (TY + 1) * TX, NB3 = TY * TX;
    for (int q = tid; q < NB1 + NB2 + NB3; q += NT) {
      if (q < NB1) {
        const int c = q % (TX + 1), r = q / (TX + 1);
        if (c > nx || r >= ny) continue;
        const double v = C[OS5 + r * 34 + c + 1] - (c2 * (SM.e3s[r + 1][c] - SM.e3s[r][c]) -
                                                   c3 * (SM.e2s[hi][r][c] - SM.e2s[lo][r][c]));
        SM.b1s[r][c] = v;
        if (c < nx || i0 + c == G.ie) {
          const int i = i0 + c;
          const int id = G.idx(k, j0 + r, i);
          if (!push || i != G.is) ST(Sout[5] + id, v);
          if (push) {
            if (i > G.is && i <= G.is + G.ng) { PMHD_CHECK_ID(G, id + G.mb[0]); ST(PL[5] + id + G.mb[0], v); }
            if (i >= G.ie - G.ng) { PMHD_CHECK_ID(G, id - G.mb[0]); ST(PR[5] + id - G.mb[0], v); }
          }
        }
      } else if (q < NB1 + NB2) {
        const int q1 = q - NB1, c = q1 % TX, r = q1 / TX;
        if (c >= nx || r > ny) continue;
        const double v = C[OS6 + r * 34 + c + 1] - (c3 * (SM.e1s[hi][r][c] - SM.e1s[lo][r][c]) -
                                                   c1 * (SM.e3s[r][c + 1] - SM.e3s[r][c]));
        SM.b2s[r][c] = v;
        if (r < ny || j0 + r == G.je) {
          const int id = G.idx(k, j0 + r, i0 + c);
          ST(Sout[6] + id, v);
          if (push) push_cell(6, i0 + c, id, v);
        }
      } else {
        const int q2 = q - NB1 - NB2, c = q2 % TX, r = q2 / TX;
        if (c >= nx || r >= ny) continue;
        const double v = C[OS7 + r * 34 + c + 1] - (c1 * (SM.e2s[hi][r][c + 1] - SM.e2s[hi][r][c]) -
                                                    c2 * (SM.e1s[hi][r + 1][c] - SM.e1s[hi][r][c]));
        SM.b3s[hi][r][c] = v;
        const int id = G.idx(k, j0 + r, i0 + c);
        ST(Sout[7] + id, SM.b3s[lo][r][c]);
        if (k + 1 == G.ke) ST(Sout[7] + id + sy, v);
        if (push) {
          push_cell(7, i0 + c, id, SM.b3s[lo][r][c]);
          if (k + 1 == G.ke) push_cell(7, i0 + c, id + sy, v);
        }
      }
    }
    __syncthreads();

    // ---- conserved update + end-of-stage cons_to_prim (threads < NC) --------
    if (own) {
      const int i = i0 + tx, j = j0 + ty;
      const int id = G.idx(k, j, i);
      PMHD_CHECK_ID(G, id + G.sy);
      double u[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double* X1 = C + OX1 + v * SX1 + ty * 34 + tx;
        const double* X2 = C + OX2 + v * SX2 + ty * 32 + tx;
        const double x3up = C[OX3 + v * SC + ty * 32 + tx];
        double du = c1 * (X1[1] - X1[0]) + c2 * (X2[32] - X2[0]);
        du = du + c3 * (x3up - x3lo[v]);
        u[v] = C[OSB + v * SSB + ty * 34 + tx + 1] - du;
        x3lo[v] = x3up;
      }
      double bc[3], w[8];
      bc[0] = 0.5 * (SM.b1s[ty][tx] + SM.b1s[ty][tx + 1]);
      bc[1] = 0.5 * (SM.b2s[ty][tx] + SM.b2s[ty + 1][tx]);
      bc[2] = 0.5 * (SM.b3s[lo][ty][tx] + SM.b3s[hi][ty][tx]);
      const int fl = cons_to_prim(u, bc, ph, w, true);
      if (fl & 3)
        atomicAdd(&red[ks.stage].floor_count, (unsigned long long)(((fl & 1) ? 1 : 0) + ((fl & 2) ? 1 : 0)));
      if (fl & 4) {
        const long long gi = (long long)B.c[0] * G.mb[0] + (i - G.is);
        const long long gj = (long long)B.c[1] * G.mb[1] + (j - G.js);
        const long long gk = (long long)B.c[2] * G.mb[2] + (k - G.ks);
        atomicMin(&red[ks.stage].bad_key, (unsigned long long)((gk * G.nx[1] + gj) * G.nx[0] + gi));
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) ST(Sout[v] + id, u[v]);
      if (push) {
#pragma unroll
        for (int v = 0; v < 5; ++v) push_cell(v, i, id, u[v]);
      }
      if (want_dt) {
#pragma unroll
        for (int v = 0; v < 8; ++v) SM.wv[v][tid] = w[v];
      }
    }
    // (also: every read of cell slot lo is done before step k+1 refills it)
    __syncthreads();
    // ---- dt terms: dx_d / (|v_d| + c_f,d), 3 per cell over all threads -------
    if (want_dt) {
      for (int q = tid; q < 3 * NC; q += NT) {
        const int cc = q % NC, dd = q / NC;
        if (cc % TX >= nx || cc / TX >= ny) continue;
        const double d = SM.wv[0][cc], p = SM.wv[4][cc];
        const int d1 = (dd == 2) ? 0 : dd + 1, d2 = (dd == 0) ? 2 : dd - 1;
        const double bn = SM.wv[5 + dd][cc], bt1 = SM.wv[5 + d1][cc], bt2 = SM.wv[5 + d2][cc];
        const double cf = fast_speed_n(d, p, bn, bt1, bt2, ph.gamma);
        const double dxd = (dd == 0) ? G.dx[0] : ((dd == 1) ? G.dx[1] : G.dx[2]);  // (no local copy of G.dx)
        tmin = fmin(tmin, ddiv(dxd, fabs(SM.wv[1 + dd][cc]) + cf));
      }
    }
  }
  if (PROF) {
    if (tid == 0) {
      SM.tph[2] += clock64() - SM.tph[0];
      atomicAdd(&red[ks.stage].phase[3], (unsigned long long)SM.tph[1]);
      atomicAdd(&red[ks.stage].phase[4], (unsigned long long)SM.tph[2]);
    }
  }
  if (want_dt) {
    for (int o = 16; o > 0; o >>= 1) tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
    if ((tid & 31) == 0) SM.redbuf[tid >> 5] = tmin;
    __syncthreads();
    if (tid < 32) {
      double v = (tid < NT / 32) ? SM.redbuf[tid] : 1.0e300;
      for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (tid == 0) atomicMin(&red[0].dt_bits, (unsigned long long)__double_as_longlong(v));
    }
  }
}

}  // namespace

int update_tma_maps_per_block() { return kMaps; }

// Box (width, height) of map id a (see the id table above).
// (box[2]: first cell relative to the tile origin i0; its address must be
// 16 B aligned, which the host checks)
void update_tma_box(int a, int box[3]) {
  box[2] = box_i(a);
  if (a < 12) { box[0] = ew(a); box[1] = EBH; }
  else if (a < 17) { box[0] = 34; box[1] = TY; }
  else if (a < 22) { box[0] = 32; box[1] = TY + 1; }
  else if (a < 27) { box[0] = 32; box[1] = TY; }
  else if (a == 33) { box[0] = 34; box[1] = TY + 1; }
  else { box[0] = 34; box[1] = TY; }
}

// The device array each map id of block B covers (st0: the table's u^n).
const double* update_tma_array(const DevBlock& B, int a) {
  if (a < 3) return B.fx[0][5 + a];
  if (a < 6) return B.fx[1][2 + a];
  if (a < 9) return B.fx[2][a - 1];
  if (a < 12) return B.ec[a - 9];
  if (a < 17) return B.fx[0][a - 12];
  if (a < 22) return B.fx[1][a - 17];
  if (a < 27) return B.fx[2][a - 22];
  return B.st[0][a - 27];  // 27..34: u^n[0..4], b1f, b2f, b3f
}

void launch_update_tma(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks,
                       const KStage* kd, DevRed* red, int want_dt, int kr0, int kr1, cudaStream_t s,
                       const CUtensorMap* maps, unsigned long long xoffm, int push) {
  // segments of 32 planes where the mesh gives >= 2 waves, else 16
  const int tiles = ((G.ie - G.is + TX - 1) / TX) * ((G.je - G.js + TY - 1) / TY) * G.nb;
  const int nk = kr1 - kr0;
  const bool long_seg = (long long)tiles * ((nk + 31) / 32) >= 2 * 148 * MINB;
  const int seg = long_seg ? 32 : 16;
  const int nseg = (nk + seg - 1) / seg;
  const dim3 grid((G.ie - G.is + TX - 1) / TX, (G.je - G.js + TY - 1) / TY, nseg * G.nb);
  constexpr int smem = (int)sizeof(TSmem) + 128;
#define PMHD_UPDATE_TMA_LAUNCH(SG)                                                                        \
  do {                                                                                                    \
    static std::atomic<unsigned long long> attr_devs{0};                                                  \
    int dev = 0;                                                                                          \
    cudaGetDevice(&dev);                                                                                  \
    if (!(attr_devs.load() & (1ULL << (dev & 63)))) {                                                     \
      cudaFuncSetAttribute(k_update_tma<SG, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);       \
      cudaFuncSetAttribute(k_update_tma<SG, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);       \
      cudaFuncSetAttribute(k_update_tma<SG, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);       \
      attr_devs.fetch_or(1ULL << (dev & 63));                                                             \
    }                                                                                                     \
    if (kd)                                                                                               \
      k_update_tma<SG, 2><<<grid, NT, smem, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, maps, xoffm, push); \
    else if (ph.prof)                                                                                     \
      k_update_tma<SG, 1><<<grid, NT, smem, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, maps, xoffm, push); \
    else                                                                                                  \
      k_update_tma<SG, 0><<<grid, NT, smem, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, maps, xoffm, push); \
  } while (0)
  if (seg == 32) PMHD_UPDATE_TMA_LAUNCH(32);
  else PMHD_UPDATE_TMA_LAUNCH(16);
#undef PMHD_UPDATE_TMA_LAUNCH
}

}  // namespace pmhd_gpu
