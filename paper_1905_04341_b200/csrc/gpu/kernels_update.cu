// kernels_update.cu -- fused end of a VL2 stage: corner EMFs (ct_emf,
// SPEC.md:191-199), constrained-transport face update (ct_update_face_b,
// SPEC.md:200-208), conserved update ("integrate"),
// face_to_center_b + end-of-stage cons_to_prim with floors / error detection
// and the compute_dt partial min
// (SPEC.md:159-167), in ONE kernel over all MeshBlocks.
//
// A CTA of 256 threads owns a 32 x 8 tile of cells in one k-plane.  It
// converts the stage-input state of the (34 x 10 x 3)-cell neighbourhood to
// the cell-centred E = -v x B in shared memory, forms every corner EMF that
// bounds its cells (reading the face E / upwind weights written by the flux
// kernels), updates every face bounding its cells (also the shared upper
// faces, which only the owner writes back), then updates and re-primitivises
// its cells.  Outputs go to a separate buffer (st[out_sel]), so tiles that
// recompute a shared face never read a value another tile has overwritten.
#include <atomic>

#include "kernels.cuh"
#include "tma.cuh"

namespace pmhd_gpu {

namespace {

#ifndef PMHD_UPDATE_UY
#define PMHD_UPDATE_UY 8  // tile rows (one thread per cell: 32 x UY threads)
#endif
constexpr int UX = 32, UY = PMHD_UPDATE_UY, UTHR = UX * UY;
constexpr int EX = UX + 2, EY = UY + 2;  // Ec box extents (cells i0-1 .. i1, j0-1 .. j1)
#ifndef PMHD_UPDATE_TMA
// 1: stream the E ring with TMA one plane ahead (measured at 256^3: -2 %
// against the plain loads -- the extra live state costs registers -- so off)
#define PMHD_UPDATE_TMA 0
#endif
// E ring slot stride (doubles): 128 B aligned for TMA boxes, dense otherwise
constexpr int ECS = PMHD_UPDATE_TMA ? ((EX * EY * 8 + 127) / 128) * 16 : EX * EY;
#ifndef PMHD_UPDATE_MINB
#define PMHD_UPDATE_MINB (1280 / (32 * PMHD_UPDATE_UY))  // 40 warps/SM of budget (48 regs)
#endif
#ifndef PMHD_UPDATE_SEG
#define PMHD_UPDATE_SEG 16  // max k planes marched by one CTA (shorter for small meshes)
#endif

// A CTA owns a 32 x 8 (i, j) column of cells and marches k through a segment
// [kb, kb + SEG).  What a plane shares with the next is carried instead of
// recomputed: the cell-centred E ring holds planes k and k+1 (one new plane
// loaded per step), E1 / E2 at k+1/2 become the k-1/2 values of the next
// step, and so does the new b3 face at k+1.
#ifndef PMHD_UPD_EC_SMEM
#define PMHD_UPD_EC_SMEM 1  // 0: read the cell-centred E through L1 instead of the shared-memory ring
#endif
#ifndef PMHD_UPD_FLAT_B
#define PMHD_UPD_FLAT_B 0  // 1: phase B (E3 + E1 + E2) as one flat item list (spills at 48 regs: 1.79 vs 1.55 ms)
#endif
#ifndef PMHD_UPD_FLAT_C
#define PMHD_UPD_FLAT_C 1  // phase C (b1 + b2 + b3) as one flat item list
#endif
#ifndef PMHD_UPDATE_STCS
#define PMHD_UPDATE_STCS 1  // streaming stores of the new state (+0.25 %)
#endif
// new state stores (streaming when PMHD_UPDATE_STCS)
__device__ __forceinline__ void ST(double* p, double v) {
#if PMHD_UPDATE_STCS
  __stcs(p, v);
#else
  *p = v;
#endif
}

// Shared memory of one CTA (dynamic: > 48 KB for 32 x 16 tiles).
struct alignas(PMHD_UPDATE_TMA ? 128 : 16) UpdSmem {
  // cell-centred E ring: [component][k & 1] boxes of EY x EX (one TMA box
  // each; slots padded to 128 B multiples)
  double ecbuf[3][2][PMHD_UPD_EC_SMEM ? ECS : 1];
  unsigned long long bar[2];    // TMA completion barriers, one per ring slot
  double e3s[UY + 1][UX + 1];   // E3 at (k, j-1/2, i-1/2)
  double e1s[2][UY + 1][UX];    // E1 at (k -/+ 1/2, j-1/2, i), slot by parity
  double e2s[2][UY][UX + 1];    // E2 at (k -/+ 1/2, j, i-1/2)
  double b1s[UY][UX + 1];
  double b2s[UY + 1][UX];
  double b3s[2][UY][UX];        // new b3 at faces k / k+1, slot by parity
  double redbuf[UTHR / 32];
  long long tph[3];             // profiling (thread 0): mark, EMF cycles, update cycles
};

// MODE: 0 product, 1 region profiling, 2 graph-replayed cycle (stage from kd)
template <int SEG, int MODE>
__global__ void __launch_bounds__(UTHR, PMHD_UPDATE_MINB)
k_update_fused(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, KStage ks_arg,
               const KStage* __restrict__ kd, DevRed* red, int want_dt, int kr0, int kr1,
               const CUtensorMap* __restrict__ ec_maps, int push) {
  // graph-replayed cycle past the end of the run: tested after the prologue's
  // E loads are issued (before any global write)
  constexpr bool PROF = (MODE == 1);
  if (MODE == 2 && kd->skip) return;  // replayed cycle past the end of the run
  const KStage ks = (MODE == 2) ? *kd : ks_arg;
  extern __shared__ __align__(16) unsigned char upd_smem[];
  // (128 B alignment for the TMA boxes; the launch adds 128 bytes of slack)
#if PMHD_UPDATE_TMA
  UpdSmem& SM = *reinterpret_cast<UpdSmem*>((reinterpret_cast<uintptr_t>(upd_smem) + 127) &
                                            ~uintptr_t(127));
#else
  UpdSmem& SM = *reinterpret_cast<UpdSmem*>(upd_smem);
#endif
  auto ec = [&](int c, int sl) { return reinterpret_cast<double(*)[EX]>(&SM.ecbuf[c][sl][0]); };
  // E of component c at E-box row r, column q of plane kk: the ring slot of
  // kk, or (PMHD_UPD_EC_SMEM=0) straight from the array through L1
  struct EcRows {
    const double* p;
    int sx;
    __device__ __forceinline__ const double* operator[](int r) const { return p + r * sx; }
  };
  auto& e3s = SM.e3s;
  auto& e1s = SM.e1s;
  auto& e2s = SM.e2s;
  auto& b1s = SM.b1s;
  auto& b2s = SM.b2s;
  auto& b3s = SM.b3s;
  auto& redbuf = SM.redbuf;
  auto& tph = SM.tph;
  if (PROF && threadIdx.x == 0) { tph[0] = clock64(); tph[1] = tph[2] = 0; }

  const bool d3 = (G.dim == 3);
  const int nseg = (kr1 - kr0 + SEG - 1) / SEG;
  const int b = blockIdx.z / nseg;
  const int kb = kr0 + (int)(blockIdx.z % nseg) * SEG;
  const int kend = min(kb + SEG, kr1);
  const int i0 = G.is + blockIdx.x * UX, j0 = G.js + blockIdx.y * UY;
  const int nx = min(UX, G.ie - i0), ny = min(UY, G.je - j0);
  const DevBlock& B = blks[b];
#if PMHD_UPD_EC_SMEM
  auto ecx = [&](int c, int kk) { return ec(c, kk & 1); };
#else
  auto ecx = [&](int c, int kk) { return EcRows{B.ec[c] + G.idx(kk, j0 - 1, i0 - 1), G.sx}; };
#endif
  double* const* Sb = B.st[0];
  double* const* Sout = B.st[ks.out_sel];
  double* const* X1 = B.fx[0];
  double* const* X2 = B.fx[1];
  double* const* X3 = B.fx[2];
  const int sx = G.sx, sy = G.sy;
  const int tid = threadIdx.x;
  const int mode = ph.emf;
  const double c1 = ks.c1, c2 = ks.c2, c3 = ks.c3;
  // x1 ghost push (all x1 neighbours local, launch flag): every value this
  // kernel writes that the x1 ghost exchange would copy is also stored at
  // its ghost position in the neighbour block, so the stage's x1 exchange
  // launch is skipped.  PL: the left neighbour (its right ghosts come from
  // cells [is, is+ng)), PR: the right neighbour (left ghosts from
  // [ie-ng, ie)); for b1f the normal-face ranges of the exchange apply, and
  // the shared face is is left to the left neighbour's ie face.
  double* const* PL = push ? blks[B.nbr[0][0]].st[ks.out_sel] : nullptr;
  double* const* PR = push ? blks[B.nbr[0][1]].st[ks.out_sel] : nullptr;
  auto push_cell = [&](int v, int i, int id, double val) {
    if (i < G.is + G.ng) { PMHD_CHECK_ID(G, id + G.mb[0]); ST(PL[v] + id + G.mb[0], val); }
    if (i >= G.ie - G.ng) { PMHD_CHECK_ID(G, id - G.mb[0]); ST(PR[v] + id - G.mb[0], val); }
  };

  // cell-centred E of plane kk (written by the last-direction flux kernel
  // from the stage-input primitives) into ring slot kk & 1
  auto load_ec = [&](int kk) {
    const int sl = kk & 1;
#pragma unroll
    for (int q = tid; q < EY * EX; q += UTHR) {
      const int c = q % EX, r = q / EX;
      if (c > nx + 1 || r > ny + 1) continue;
      const int id = G.idx(kk, j0 - 1 + r, i0 - 1 + c);
      PMHD_CHECK_ID(G, id);
      ec(0, sl)[r][c] = __ldg(B.ec[0] + id);
      ec(1, sl)[r][c] = __ldg(B.ec[1] + id);
      ec(2, sl)[r][c] = __ldg(B.ec[2] + id);
    }
  };
  // E1 / E2 on the edge plane kk - 1/2 (3D; in 2D the face E of plane k)
  // into slot h
  auto edge_emfs = [&](int kk, int h) {
    const int pa = kk & 1, pm = (kk - 1) & 1;  // Ec slots of kk and kk-1
#pragma unroll
    for (int q = tid; q < (UY + 1) * UX; q += UTHR) {
      const int c = q % UX, r = q / UX;
      if (c >= nx || r > ny) continue;
      const int id = G.idx(d3 ? kk : kb, j0 + r, i0 + c);
      if (d3) PMHD_CHECK_ID(G, id - G.sy);
      PMHD_CHECK_ID(G, id);
      double e;
      if (d3) {
        e = corner_emf(mode, X2[5][id], X2[5][id - sy], X3[6][id], X3[6][id - sx], X2[7][id],
                       X2[7][id - sy], X3[7][id], X3[7][id - sx], ecx(0, kk)[r + 1][c + 1],
                       ecx(0, kk)[r][c + 1], ecx(0, kk - 1)[r + 1][c + 1], ecx(0, kk - 1)[r][c + 1]);
      } else {
        e = X2[5][id];
      }
      e1s[h][r][c] = e;
    }
#pragma unroll
    for (int q = tid; q < UY * (UX + 1); q += UTHR) {
      const int c = q % (UX + 1), r = q / (UX + 1);
      if (c > nx || r >= ny) continue;
      const int id = G.idx(d3 ? kk : kb, j0 + r, i0 + c);
      double e;
      if (d3) {
        e = corner_emf(mode, X3[5][id], X3[5][id - 1], X1[6][id], X1[6][id - sy], X3[7][id],
                       X3[7][id - 1], X1[7][id], X1[7][id - sy], ecx(1, kk)[r + 1][c + 1],
                       ecx(1, kk - 1)[r + 1][c + 1], ecx(1, kk)[r + 1][c], ecx(1, kk - 1)[r + 1][c]);
      } else {
        e = X1[6][id];
      }
      e2s[h][r][c] = e;
    }
  };
  // Phase B of step k as ONE flat item list (E3 at plane k, then E1 and E2
  // at k + 1/2 into slot hi), so the 256 threads take ceil(849 / 256) = 4
  // passes instead of 2 + 2 + 2 with three separate loops; same operands
  // and expressions as the loops above (3D only).
  constexpr int NE3 = (UY + 1) * (UX + 1), NE1 = (UY + 1) * UX, NE2 = UY * (UX + 1);
  auto emf_items = [&](int k, int lo, int hi) {
    const int kk = k + 1;
    for (int q = tid; q < NE3 + NE1 + NE2; q += UTHR) {
      if (q < NE3) {
        const int c = q % (UX + 1), r = q / (UX + 1);
        if (c > nx || r > ny) continue;
        const int id = G.idx(k, j0 + r, i0 + c);
        PMHD_CHECK_ID(G, id - G.sx);
        const int ec_c = c + 1, ec_r = r + 1;
        e3s[r][c] = corner_emf(mode, X1[5][id], X1[5][id - sx], X2[6][id], X2[6][id - 1], X1[7][id],
                               X1[7][id - sx], X2[7][id], X2[7][id - 1], ecx(2, k)[ec_r][ec_c],
                               ecx(2, k)[ec_r][ec_c - 1], ecx(2, k)[ec_r - 1][ec_c],
                               ecx(2, k)[ec_r - 1][ec_c - 1]);
      } else if (q < NE3 + NE1) {
        const int q1 = q - NE3, c = q1 % UX, r = q1 / UX;
        if (c >= nx || r > ny) continue;
        const int id = G.idx(kk, j0 + r, i0 + c);
        PMHD_CHECK_ID(G, id - G.sy);
        PMHD_CHECK_ID(G, id);
        e1s[hi][r][c] = corner_emf(mode, X2[5][id], X2[5][id - sy], X3[6][id], X3[6][id - sx], X2[7][id],
                                   X2[7][id - sy], X3[7][id], X3[7][id - sx], ecx(0, kk)[r + 1][c + 1],
                                   ecx(0, kk)[r][c + 1], ecx(0, k)[r + 1][c + 1], ecx(0, k)[r][c + 1]);
      } else {
        const int q2 = q - NE3 - NE1, c = q2 % (UX + 1), r = q2 / (UX + 1);
        if (c > nx || r >= ny) continue;
        const int id = G.idx(kk, j0 + r, i0 + c);
        e2s[hi][r][c] = corner_emf(mode, X3[5][id], X3[5][id - 1], X1[6][id], X1[6][id - sy], X3[7][id],
                                   X3[7][id - 1], X1[7][id], X1[7][id - sy], ecx(1, kk)[r + 1][c + 1],
                                   ecx(1, k)[r + 1][c + 1], ecx(1, kk)[r + 1][c], ecx(1, k)[r + 1][c]);
      }
    }
  };
  // new b3 on face plane kk from the edge EMFs in slot h
  auto face_b3 = [&](int kk, int h) {
#pragma unroll
    for (int q = tid; q < UY * UX; q += UTHR) {
      const int c = q % UX, r = q / UX;
      if (c >= nx || r >= ny) continue;
      const int id = G.idx(kk, j0 + r, i0 + c);
      PMHD_CHECK_ID(G, id);
      const double v = Sb[7][id] - (c1 * (e2s[h][r][c + 1] - e2s[h][r][c]) -
                                    c2 * (e1s[h][r + 1][c] - e1s[h][r][c]));
      b3s[h][r][c] = v;
    }
  };

  // TMA E ring (3D): thread 0 issues plane kk into its slot (one box per
  // component); everyone waits on the slot's barrier before reading it.  A
  // plane is issued one step ahead, as soon as its slot's previous plane has
  // been read, so the E stream overlaps the CT / update phases.
#if PMHD_UPDATE_TMA
  const bool tma = (ec_maps != nullptr) && d3;
#else
  constexpr bool tma = false;
#endif
  unsigned eph = 0u;  // barrier phase bit of each ring slot (bit sl)
  auto issue_ec = [&](int kk) {
    if (tid == 0) {
      const int sl = kk & 1;
      fence_proxy_async_smem();  // after the generic reads of the slot
      mbar_expect_tx(&SM.bar[sl], 3u * EX * EY * 8u);
      for (int c = 0; c < 3; ++c)  // the maps start at i = -1: cell i0-1 is x = i0
        tma_load_3d(&SM.ecbuf[c][sl][0], ec_maps + 3 * b + c, &SM.bar[sl], i0, j0 - 1, kk);
    }
  };
  auto wait_ec = [&](int kk) {
    const int sl = kk & 1;
    mbar_wait(&SM.bar[sl], (eph >> sl) & 1u);
    eph ^= 1u << sl;
  };

  // ---- prologue: Ec planes kb-1, kb and the edge EMFs at kb - 1/2 ----------
  if (tma) {
    if (tid == 0) {
      mbar_init(&SM.bar[0], 1);
      mbar_init(&SM.bar[1], 1);
      mbar_init_fence();
    }
    __syncthreads();
    issue_ec(kb - 1);
    issue_ec(kb);
    wait_ec(kb - 1);
    wait_ec(kb);
  } else {
    if (PMHD_UPD_EC_SMEM) {
      if (d3) load_ec(kb - 1);
      load_ec(kb);
    }
  }
  __syncthreads();
  edge_emfs(kb, kb & 1);
  __syncthreads();
  if (tma && kb + 1 <= kend) issue_ec(kb + 1);  // (slot of kb-1, read by the edge EMFs above)
  face_b3(kb, kb & 1);

#ifdef PMHD_DIAG_UPD_NO_D
  double tmin = 1.0e-5;
#else
  double tmin = 1.0e300;
#endif
  for (int k = kb; k < kend; ++k) {
    const int lo = k & 1, hi = lo ^ 1;  // slots of k - 1/2 and k + 1/2
    if (PROF && tid == 0 && k > kb) { const long long t = clock64(); tph[2] += t - tph[0]; tph[0] = t; }
    // ---- A: the next Ec plane (slot of k-1, no longer needed) --------------
    if (tma) wait_ec(k + 1);
    else if (PMHD_UPD_EC_SMEM && d3) load_ec(k + 1);
    __syncthreads();
    // ---- B: E3 at plane k, E1 / E2 at k + 1/2 -------------------------------
    if (PMHD_UPD_FLAT_B && d3) emf_items(k, lo, hi);
    else {
#pragma unroll
    for (int q = tid; q < (UY + 1) * (UX + 1); q += UTHR) {
      const int c = q % (UX + 1), r = q / (UX + 1);
      if (c > nx || r > ny) continue;
      const int id = G.idx(k, j0 + r, i0 + c);
      PMHD_CHECK_ID(G, id - G.sx);
      const int ec_c = c + 1, ec_r = r + 1;
      e3s[r][c] = corner_emf(mode, X1[5][id], X1[5][id - sx], X2[6][id], X2[6][id - 1], X1[7][id],
                             X1[7][id - sx], X2[7][id], X2[7][id - 1], ecx(2, k)[ec_r][ec_c],
                             ecx(2, k)[ec_r][ec_c - 1], ecx(2, k)[ec_r - 1][ec_c],
                             ecx(2, k)[ec_r - 1][ec_c - 1]);
    }
    edge_emfs(k + 1, hi);
    }
    __syncthreads();
    if (tma && k + 2 <= kend) issue_ec(k + 2);  // into slot lo: plane k was last read just above
    if (PROF && tid == 0) { const long long t = clock64(); tph[1] += t - tph[0]; tph[0] = t; }
#if PMHD_UPD_FLAT_C
    // ---- C: constrained-transport face update: b1f (faces i0 .. i0+nx),
    // b2f (faces j0 .. j0+ny) and b3f at face k + 1 (face k carried) as one
    // flat item list (4 passes of the 256 threads instead of 2 + 2 + 1)
    constexpr int NB1 = UY * (UX + 1), NB2 = (UY + 1) * UX, NB3 = UY * UX;
    for (int q = tid; q < NB1 + NB2 + NB3; q += UTHR) {
      if (q < NB1) {
        const int c = q % (UX + 1), r = q / (UX + 1);
        if (c > nx || r >= ny) continue;
        const int id = G.idx(k, j0 + r, i0 + c);
        double v;
        if (d3) v = Sb[5][id] - (c2 * (e3s[r + 1][c] - e3s[r][c]) - c3 * (e2s[hi][r][c] - e2s[lo][r][c]));
        else v = Sb[5][id] - c2 * (e3s[r + 1][c] - e3s[r][c]);
        b1s[r][c] = v;
        if (c < nx || i0 + c == G.ie) {
          const int i = i0 + c;
          if (!push || i != G.is) ST(Sout[5] + id, v);
          if (push) {
            if (i > G.is && i <= G.is + G.ng) { PMHD_CHECK_ID(G, id + G.mb[0]); ST(PL[5] + id + G.mb[0], v); }
            if (i >= G.ie - G.ng) { PMHD_CHECK_ID(G, id - G.mb[0]); ST(PR[5] + id - G.mb[0], v); }
          }
        }
      } else if (q < NB1 + NB2) {
        const int q1 = q - NB1, c = q1 % UX, r = q1 / UX;
        if (c >= nx || r > ny) continue;
        const int id = G.idx(k, j0 + r, i0 + c);
        double v;
        if (d3) v = Sb[6][id] - (c3 * (e1s[hi][r][c] - e1s[lo][r][c]) - c1 * (e3s[r][c + 1] - e3s[r][c]));
        else v = Sb[6][id] + c1 * (e3s[r][c + 1] - e3s[r][c]);
        b2s[r][c] = v;
        if (r < ny || j0 + r == G.je) {
          ST(Sout[6] + id, v);
          if (push) push_cell(6, i0 + c, id, v);
        }
      } else {  // face_b3(k + 1, hi) and the store of face k
        const int q2 = q - NB1 - NB2, c = q2 % UX, r = q2 / UX;
        if (c >= nx || r >= ny) continue;
        const int id = G.idx(k, j0 + r, i0 + c);
        PMHD_CHECK_ID(G, id + sy);
        const double v = Sb[7][id + sy] - (c1 * (e2s[hi][r][c + 1] - e2s[hi][r][c]) -
                                          c2 * (e1s[hi][r + 1][c] - e1s[hi][r][c]));
        b3s[hi][r][c] = v;
        ST(Sout[7] + id, b3s[lo][r][c]);
        if (k + 1 == G.ke) ST(Sout[7] + id + sy, v);
        if (push) {
          push_cell(7, i0 + c, id, b3s[lo][r][c]);
          if (k + 1 == G.ke) push_cell(7, i0 + c, id + sy, v);
        }
      }
    }
#else
    // ---- C: constrained-transport face update -------------------------------
    for (int q = tid; q < UY * (UX + 1); q += UTHR) {  // b1f, faces i0 .. i0+nx
      const int c = q % (UX + 1), r = q / (UX + 1);
      if (c > nx || r >= ny) continue;
      const int id = G.idx(k, j0 + r, i0 + c);
      double v;
      if (d3) v = Sb[5][id] - (c2 * (e3s[r + 1][c] - e3s[r][c]) - c3 * (e2s[hi][r][c] - e2s[lo][r][c]));
      else v = Sb[5][id] - c2 * (e3s[r + 1][c] - e3s[r][c]);
      b1s[r][c] = v;
      if (c < nx || i0 + c == G.ie) {
        const int i = i0 + c;
        if (!push || i != G.is) ST(Sout[5] + id, v);
        if (push) {
          if (i > G.is && i <= G.is + G.ng) { PMHD_CHECK_ID(G, id + G.mb[0]); ST(PL[5] + id + G.mb[0], v); }
          if (i >= G.ie - G.ng) { PMHD_CHECK_ID(G, id - G.mb[0]); ST(PR[5] + id - G.mb[0], v); }
        }
      }
    }
    for (int q = tid; q < (UY + 1) * UX; q += UTHR) {  // b2f, faces j0 .. j0+ny
      const int c = q % UX, r = q / UX;
      if (c >= nx || r > ny) continue;
      const int id = G.idx(k, j0 + r, i0 + c);
      double v;
      if (d3) v = Sb[6][id] - (c3 * (e1s[hi][r][c] - e1s[lo][r][c]) - c1 * (e3s[r][c + 1] - e3s[r][c]));
      else v = Sb[6][id] + c1 * (e3s[r][c + 1] - e3s[r][c]);
      b2s[r][c] = v;
      if (r < ny || j0 + r == G.je) {
        ST(Sout[6] + id, v);
        if (push) push_cell(6, i0 + c, id, v);
      }
    }
    face_b3(k + 1, hi);  // b3 at face k + 1 (face k carried)
    {
      const int c = tid % UX, r = tid / UX;
      if (c < nx && r < ny) {
        const int id = G.idx(k, j0 + r, i0 + c);
        ST(Sout[7] + id, b3s[lo][r][c]);
        if (k + 1 == G.ke) ST(Sout[7] + id + sy, b3s[hi][r][c]);
        if (push) {
          push_cell(7, i0 + c, id, b3s[lo][r][c]);
          if (k + 1 == G.ke) push_cell(7, i0 + c, id + sy, b3s[hi][r][c]);
        }
      }
    }
#endif
    __syncthreads();

    // ---- D: conserved update + end-of-stage cons_to_prim + dt --------------
    {
      const int c = tid % UX, r = tid / UX;
#ifdef PMHD_DIAG_UPD_NO_D  // diagnostic (never shipped): EMF + CT phases + a state copy only
      if (c < nx && r < ny) {
        const int id = G.idx(k, j0 + r, i0 + c);
#pragma unroll
        for (int v = 0; v < 5; ++v) ST(Sout[v] + id, Sb[v][id]);
      }
      if (false) {
#else
      if (c < nx && r < ny) {
#endif
        const int i = i0 + c, j = j0 + r;
        const int id = G.idx(k, j, i);
        PMHD_CHECK_ID(G, id + G.sy);
        double u[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
#if PMHD_DIAG_UPD_DU == 1  // diagnostic (never shipped): one flux load per direction
          double du = 1e-30 * (c1 * X1[v][id] + c2 * X2[v][id] + c3 * X3[v][id]);
#elif PMHD_DIAG_UPD_DU == 2  // diagnostic: no flux loads
          double du = 0.0;
#else
          double du = c1 * (X1[v][id + 1] - X1[v][id]) + c2 * (X2[v][id + sx] - X2[v][id]);
          if (d3) du = du + c3 * (X3[v][id + sy] - X3[v][id]);
#endif
          u[v] = Sb[v][id] - du;
        }
        double bc[3], w[8];
        bc[0] = 0.5 * (b1s[r][c] + b1s[r][c + 1]);
        bc[1] = 0.5 * (b2s[r][c] + b2s[r + 1][c]);
        bc[2] = 0.5 * (b3s[lo][r][c] + b3s[hi][r][c]);
        const int fl = cons_to_prim(u, bc, ph, w, true);
        if (fl & 3)
          atomicAdd(&red[ks.stage].floor_count,
                    (unsigned long long)(((fl & 1) ? 1 : 0) + ((fl & 2) ? 1 : 0)));
        if (fl & 4) {
          const long long gi = (long long)B.c[0] * G.mb[0] + (i - G.is);
          const long long gj = (long long)B.c[1] * G.mb[1] + (j - G.js);
          const long long gk = d3 ? (long long)B.c[2] * G.mb[2] + (k - G.ks) : 0;
          atomicMin(&red[ks.stage].bad_key, (unsigned long long)((gk * G.nx[1] + gj) * G.nx[0] + gi));
        }
#pragma unroll
        for (int v = 0; v < 5; ++v) ST(Sout[v] + id, u[v]);
        if (push) {
#pragma unroll
          for (int v = 0; v < 5; ++v) push_cell(v, i, id, u[v]);
        }
        if (want_dt) {
          const double d = w[0], p = w[4];
          const double cf1 = fast_speed_n(d, p, w[5], w[6], w[7], ph.gamma);
          const double cf2 = fast_speed_n(d, p, w[6], w[7], w[5], ph.gamma);
          double t = fmin(ddiv(G.dx[0], fabs(w[1]) + cf1), ddiv(G.dx[1], fabs(w[2]) + cf2));
          if (d3) {
            const double cf3 = fast_speed_n(d, p, w[7], w[5], w[6], ph.gamma);
            t = fmin(t, ddiv(G.dx[2], fabs(w[3]) + cf3));
          }
          tmin = fmin(tmin, t);
        }
      }
    }
  }
  if (PROF) {
    __syncthreads();
    if (tid == 0) {
      tph[2] += clock64() - tph[0];
      atomicAdd(&red[ks.stage].phase[3], (unsigned long long)tph[1]);
      atomicAdd(&red[ks.stage].phase[4], (unsigned long long)tph[2]);
    }
  }
  if (want_dt) {
    for (int o = 16; o > 0; o >>= 1) tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
    if ((tid & 31) == 0) redbuf[tid >> 5] = tmin;
    __syncthreads();
    if (tid < 32) {
      double v = (tid < UTHR / 32) ? redbuf[tid] : 1.0e300;
      for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (tid == 0) atomicMin(&red[0].dt_bits, (unsigned long long)__double_as_longlong(v));
    }
  }
}

}  // namespace

void update_ec_box(int box[2]) {
  box[0] = EX;
  box[1] = EY;
}

bool update_uses_tma() { return PMHD_UPDATE_TMA != 0; }

void launch_update_fused(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks,
                         const KStage* kd, DevRed* red, int want_dt, int kr0, int kr1, cudaStream_t s,
                         const CUtensorMap* ec_maps, int push) {
  // segment length: PMHD_UPDATE_SEG planes, or 4 / 1 when the mesh is too
  // small to fill ~2 waves of 148 SMs x 5 CTAs otherwise
  const int tiles = ((G.ie - G.is + UX - 1) / UX) * ((G.je - G.js + UY - 1) / UY) * G.nb;
  const int nk = kr1 - kr0;
  const int want = (2 * 148 * PMHD_UPDATE_MINB + tiles - 1) / tiles;  // segments per column
  const int fit = (nk + want - 1) / want;                              // planes per segment
  const int seg = (fit >= PMHD_UPDATE_SEG) ? PMHD_UPDATE_SEG : (fit >= 4 ? 4 : 1);
  const int nseg = (nk + seg - 1) / seg;
  const dim3 grid((G.ie - G.is + UX - 1) / UX, (G.je - G.js + UY - 1) / UY, nseg * G.nb);
  constexpr int smem = (int)sizeof(UpdSmem) + 128;  // + alignment slack
#define PMHD_UPDATE_LAUNCH(SG)                                                                          \
  do {                                                                                                  \
    /* per device (the attribute is per-device state); atomic: contexts may  \
       live on different host threads; setting it twice is harmless */       \
    static std::atomic<unsigned long long> attr_devs{0};                                                \
    int dev = 0;                                                                                        \
    cudaGetDevice(&dev);                                                                                \
    if (!(attr_devs.load() & (1ULL << (dev & 63)))) {                                                   \
      cudaFuncSetAttribute(k_update_fused<SG, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);   \
      cudaFuncSetAttribute(k_update_fused<SG, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);   \
      cudaFuncSetAttribute(k_update_fused<SG, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);   \
      attr_devs.fetch_or(1ULL << (dev & 63));                                                           \
    }                                                                                                   \
    if (kd)                                                                                             \
      k_update_fused<SG, 2><<<grid, UTHR, smem, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, ec_maps, push);      \
    else if (ph.prof)                                                                                   \
      k_update_fused<SG, 1><<<grid, UTHR, smem, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, ec_maps, push);      \
    else                                                                                                \
      k_update_fused<SG, 0><<<grid, UTHR, smem, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, ec_maps, push);      \
  } while (0)
  if (seg == PMHD_UPDATE_SEG) PMHD_UPDATE_LAUNCH(PMHD_UPDATE_SEG);
  else if (seg == 4) PMHD_UPDATE_LAUNCH(4);
  else PMHD_UPDATE_LAUNCH(1);
#undef PMHD_UPDATE_LAUNCH
}

}  // namespace pmhd_gpu
