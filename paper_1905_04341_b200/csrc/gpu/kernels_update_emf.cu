// kernels_update_emf.cu -- the end of a VL2 stage as two barrier-free
// kernels (the default; PMHD_UPDATE=ldg selects k_update_fused), with the
// same operations and operand order as k_update_fused (kernels_update.cu),
// so the parity build is bit-identical to it and to the oracle:
//   k_edge_emf    corner EMFs E1, E2, E3 (ct_emf) into three
//                 scratch arrays (the block's primitive arrays w[0..2], which
//                 only the split debug variant uses);
//   k_cell_update constrained-transport faces (ct_update_face_b,
//                 SPEC.md:200-208), conserved update,
//                 face_to_center_b + cons_to_prim with floors / errors and
//                 the dt partial min, one thread per (i, j) column.
// Both march k with one thread per column and carry what plane k shares with
// plane k+1 in registers; no shared memory, no barriers.  In 2D
// k_edge_emf2d forms E3 only (E1 / E2 are the face values themselves).
// Measurements: DESIGN.md section 4a ("Two-kernel stage update").
#include "kernels.cuh"

namespace pmhd_gpu {

namespace {

#ifndef PMHD_EMF_CY
#define PMHD_EMF_CY 4
#endif
constexpr int CX = 32, CY = PMHD_EMF_CY, CTHR = CX * CY;  // thread columns per CTA (i, j)
#ifndef PMHD_EMF_SEG
#define PMHD_EMF_SEG 16  // edge / cell planes marched by one CTA
#endif
#ifndef PMHD_EMF_MINB
#define PMHD_EMF_MINB 10
#endif
#ifndef PMHD_CELL_MINB
#define PMHD_CELL_MINB 8
#endif
#ifndef PMHD_CELL_CARRY_E
#define PMHD_CELL_CARRY_E 0  // carry E1 / E2 of edge plane k+1 to the next cell plane in registers
#endif
#ifndef PMHD_CELL_CARRY_X3
#define PMHD_CELL_CARRY_X3 1  // carry the x3 fluxes of face k+1 to the next cell plane (+1 %, despite spills)
#endif

__device__ __forceinline__ void STC(double* p, double v) { __stcs(p, v); }

// Corner EMFs of thread column (i, j), i in [is, ie], j in [js, je]: E1 at
// edge (i, j-1/2, kk-1/2) and E2 at (i-1/2, j, kk-1/2) for edge planes kk in
// [kr0, kr1], E3 at (i-1/2, j-1/2, k) for cell planes k in [kr0, kr1), each
// stored at idx(kk, j, i) of w[0], w[1], w[2].  Plane kk-1's x2 ey / weight,
// x1 ez / weight and cell-centred E are carried from the previous step.
//
// rim (every neighbour on this rank): the block's upper rim edges (i = ie,
// j = je and, bit 1, kk = ke) are not formed here but stored by the upper
// neighbour's threads on its lower rim (i = is, j = js, kk = ks), which form
// the same edge from bit-identical operands (halo faces and cell E are exact
// images of the neighbour's own), so the grid covers the owned range only.
template <int SEG>
__global__ void __launch_bounds__(CTHR, PMHD_EMF_MINB)
k_edge_emf(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, const KStage* __restrict__ kd, int kr0,
           int kr1, int rim) {
  if (kd != nullptr && kd->skip) return;
  const int kext = (rim & 2) ? kr1 : kr1 + 1;  // edge planes [kr0, kext)
  const int nseg = (kext - kr0 + SEG - 1) / SEG;
  const int b = blockIdx.z / nseg;
  const int kb = kr0 + (int)(blockIdx.z % nseg) * SEG;
  const int kend = min(kb + SEG, kext);
  const int i = G.is + blockIdx.x * CX + threadIdx.x % CX;
  const int j = G.js + blockIdx.y * CY + threadIdx.x / CX;
  const int r1 = rim & 1;
  if (i > G.ie - r1 || j > G.je - r1) return;
  const DevBlock& B = blks[b];
  const double* __restrict__ X1e = B.fx[0][5];
  const double* __restrict__ X1b = B.fx[0][6];
  const double* __restrict__ X1w = B.fx[0][7];
  const double* __restrict__ X2e = B.fx[1][5];
  const double* __restrict__ X2b = B.fx[1][6];
  const double* __restrict__ X2w = B.fx[1][7];
  const double* __restrict__ X3e = B.fx[2][5];
  const double* __restrict__ X3b = B.fx[2][6];
  const double* __restrict__ X3w = B.fx[2][7];
  const double* __restrict__ Ec0 = B.ec[0];
  const double* __restrict__ Ec1 = B.ec[1];
  const double* __restrict__ Ec2 = B.ec[2];
  double* __restrict__ W1 = B.w[0];
  double* __restrict__ W2 = B.w[1];
  double* __restrict__ W3 = B.w[2];
  const int sx = G.sx, sy = G.sy, mode = ph.emf;
  int id = G.idx(kb, j, i);
  PMHD_CHECK_ID(G, id - sy - sx - 1);
  // plane kb-1: E1's x2 ey / weight, E2's x1 ez / weight, Ec0 at rows j, j-1
  // and Ec1 at columns i, i-1
  double a = X2e[id - sy], aw = X2w[id - sy];
  double c = X1b[id - sy], cw = X1w[id - sy];
  double e0 = Ec0[id - sy], e0m = Ec0[id - sy - sx];
  double e1 = Ec1[id - sy], e1m = Ec1[id - sy - 1];
  for (int kk = kb; kk < kend; ++kk, id += sy) {
    PMHD_CHECK_ID(G, id);
    const double an = X2e[id], awn = X2w[id];
    const double cn = X1b[id], cwn = X1w[id];
    const double e0n = Ec0[id], e0mn = Ec0[id - sx];
    const double e1n = Ec1[id], e1mn = Ec1[id - 1];
    double v1 = 0.0, v2 = 0.0, v3 = 0.0;
    if (i < G.ie) {
      v1 = corner_emf(mode, an, a, X3b[id], X3b[id - sx], awn, aw, X3w[id], X3w[id - sx], e0n, e0mn, e0, e0m);
      STC(W1 + id, v1);
    }
    if (j < G.je) {
      v2 = corner_emf(mode, X3e[id], X3e[id - 1], cn, c, X3w[id], X3w[id - 1], cwn, cw, e1n, e1, e1mn, e1m);
      STC(W2 + id, v2);
    }
    if (kk < kr1) {
      v3 = corner_emf(mode, X1e[id], X1e[id - sx], X2b[id], X2b[id - 1], cwn, X1w[id - sx], awn, X2w[id - 1],
                      Ec2[id], Ec2[id - 1], Ec2[id - sx], Ec2[id - sx - 1]);
      STC(W3 + id, v3);
    }
    // lower-rim edges are also the lower neighbours' upper-rim edges
    if (r1 && (i == G.is || j == G.js)) {
      const int oi = G.mb[0], oj = G.mb[1] * sx;
      if (i == G.is) {
        const DevBlock& L = blks[B.nbr[0][0]];
        STC(L.w[1] + id + oi, v2);
        if (kk < kr1) STC(L.w[2] + id + oi, v3);
        if (j == G.js && kk < kr1) STC(blks[L.nbr[1][0]].w[2] + id + oi + oj, v3);
      }
      if (j == G.js) {
        const DevBlock& D = blks[B.nbr[1][0]];
        STC(D.w[0] + id + oj, v1);
        if (kk < kr1) STC(D.w[2] + id + oj, v3);
      }
    }
    if ((rim & 2) && kk == G.ks) {
      const int ok = G.mb[2] * sy;
      const DevBlock& K = blks[B.nbr[2][0]];
      STC(K.w[0] + id + ok, v1);
      STC(K.w[1] + id + ok, v2);
      if (i == G.is) STC(blks[blks[B.nbr[0][0]].nbr[2][0]].w[1] + id + G.mb[0] + ok, v2);
      if (j == G.js) STC(blks[blks[B.nbr[1][0]].nbr[2][0]].w[0] + id + G.mb[1] * sx + ok, v1);
    }
    a = an; aw = awn; c = cn; cw = cwn;
    e0 = e0n; e0m = e0mn; e1 = e1n; e1m = e1mn;
  }
}

// 2D: E3 of the one cell plane; E1 / E2 are the x2 / x1 face values
// themselves (the cell kernel reads them from the face arrays).  Rim stores
// as k_edge_emf.
__global__ void __launch_bounds__(CTHR, PMHD_EMF_MINB)
k_edge_emf2d(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, const KStage* __restrict__ kd, int rim) {
  if (kd != nullptr && kd->skip) return;
  const int b = blockIdx.z;
  const int i = G.is + blockIdx.x * CX + threadIdx.x % CX;
  const int j = G.js + blockIdx.y * CY + threadIdx.x / CX;
  const int r1 = rim & 1;
  if (i > G.ie - r1 || j > G.je - r1) return;
  const DevBlock& B = blks[b];
  const int sx = G.sx, id = G.idx(G.ks, j, i);
  PMHD_CHECK_ID(G, id - sx - 1);
  const double* __restrict__ X1e = B.fx[0][5];
  const double* __restrict__ X1w = B.fx[0][7];
  const double* __restrict__ X2b = B.fx[1][6];
  const double* __restrict__ X2w = B.fx[1][7];
  const double* __restrict__ Ec2 = B.ec[2];
  const double v3 = corner_emf(ph.emf, X1e[id], X1e[id - sx], X2b[id], X2b[id - 1], X1w[id], X1w[id - sx],
                               X2w[id], X2w[id - 1], Ec2[id], Ec2[id - 1], Ec2[id - sx], Ec2[id - sx - 1]);
  STC(B.w[2] + id, v3);
  if (r1 && (i == G.is || j == G.js)) {
    const int oi = G.mb[0], oj = G.mb[1] * sx;
    if (i == G.is) {
      const DevBlock& L = blks[B.nbr[0][0]];
      STC(L.w[2] + id + oi, v3);
      if (j == G.js) STC(blks[L.nbr[1][0]].w[2] + id + oi + oj, v3);
    }
    if (j == G.js) STC(blks[B.nbr[1][0]].w[2] + id + oj, v3);
  }
}

// CT faces, conserved update, cons_to_prim and dt of thread column (i, j),
// i in [is, ie), j in [js, je), cell planes [kr0, kr1).  The column's lower
// faces (and, on the block's upper rim, its upper faces) are stored; the
// upper faces are also formed here for the cell-centred field.  b3 at face
// k+1 is carried to the next plane.
template <int SEG, bool D3>
__global__ void __launch_bounds__(CTHR, PMHD_CELL_MINB)
k_cell_update(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, KStage ks_arg,
              const KStage* __restrict__ kd, DevRed* red, int want_dt, int kr0, int kr1, int push) {
  if (kd != nullptr && kd->skip) return;
  const KStage ks = (kd != nullptr) ? *kd : ks_arg;
  __shared__ double redbuf[CTHR / 32];
  const int nseg = (kr1 - kr0 + SEG - 1) / SEG;
  const int b = blockIdx.z / nseg;
  const int kb = kr0 + (int)(blockIdx.z % nseg) * SEG;
  const int kend = min(kb + SEG, kr1);
  const int tid = threadIdx.x;
  const int i = G.is + blockIdx.x * CX + tid % CX;
  const int j = G.js + blockIdx.y * CY + tid / CX;
  const bool act = (i < G.ie && j < G.je);
  double tmin = 1.0e300;
  if (act) {
    const DevBlock& B = blks[b];
    double* const* Sb = B.st[0];
    double* const* Sout = B.st[ks.out_sel];
    double* const* X1 = B.fx[0];
    double* const* X2 = B.fx[1];
    double* const* X3 = B.fx[2];
    // E1 / E2: the edge arrays (3D) or, in 2D, the x2 / x1 face values
    const double* __restrict__ E1 = D3 ? B.w[0] : B.fx[1][5];
    const double* __restrict__ E2 = D3 ? B.w[1] : B.fx[0][6];
    const double* __restrict__ E3 = B.w[2];
    double* const* PL = push ? blks[B.nbr[0][0]].st[ks.out_sel] : nullptr;
    double* const* PR = push ? blks[B.nbr[0][1]].st[ks.out_sel] : nullptr;
    const int sx = G.sx, sy = G.sy, mb0 = G.mb[0];
    const double c1 = ks.c1, c2 = ks.c2, c3 = ks.c3;
    auto push_cell = [&](int v, int id, double val) {
      if (i < G.is + G.ng) { PMHD_CHECK_ID(G, id + mb0); STC(PL[v] + id + mb0, val); }
      if (i >= G.ie - G.ng) { PMHD_CHECK_ID(G, id - mb0); STC(PR[v] + id - mb0, val); }
    };
    int id = G.idx(kb, j, i);
    // b3 at face kb (face k is carried as the previous plane's upper face)
    double b3lo = Sb[7][id] - (c1 * (E2[id + 1] - E2[id]) - c2 * (E1[id + sx] - E1[id]));
#if PMHD_CELL_CARRY_E
    double q2 = E2[id], q2p = E2[id + 1], q1 = E1[id], q1p = E1[id + sx];  // edge plane k
#endif
#if PMHD_CELL_CARRY_X3
    double f3[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) f3[v] = D3 ? X3[v][id] : 0.0;
#endif
    for (int k = kb; k < kend; ++k, id += sy) {
      PMHD_CHECK_ID(G, id + sy + sx + 1);
#if PMHD_CELL_CARRY_E
      const double n2 = E2[id + sy], n2p = E2[id + 1 + sy], n1 = E1[id + sy], n1p = E1[id + sx + sy];
#else
      const double q2 = E2[id], q2p = E2[id + 1], q1 = E1[id], q1p = E1[id + sx];
      // edge plane k+1 (2D: both b3 layers use the plane-k edges)
      const double n2 = D3 ? E2[id + sy] : q2, n2p = D3 ? E2[id + 1 + sy] : q2p;
      const double n1 = D3 ? E1[id + sy] : q1, n1p = D3 ? E1[id + sx + sy] : q1p;
#endif
      double b1lo, b1hi, b2lo, b2hi;
      if (D3) {
        b1lo = Sb[5][id] - (c2 * (E3[id + sx] - E3[id]) - c3 * (n2 - q2));
        b1hi = Sb[5][id + 1] - (c2 * (E3[id + 1 + sx] - E3[id + 1]) - c3 * (n2p - q2p));
        b2lo = Sb[6][id] - (c3 * (n1 - q1) - c1 * (E3[id + 1] - E3[id]));
        b2hi = Sb[6][id + sx] - (c3 * (n1p - q1p) - c1 * (E3[id + sx + 1] - E3[id + sx]));
      } else {
        b1lo = Sb[5][id] - c2 * (E3[id + sx] - E3[id]);
        b1hi = Sb[5][id + 1] - c2 * (E3[id + 1 + sx] - E3[id + 1]);
        b2lo = Sb[6][id] + c1 * (E3[id + 1] - E3[id]);
        b2hi = Sb[6][id + sx] + c1 * (E3[id + sx + 1] - E3[id + sx]);
      }
      const double b3hi = Sb[7][id + sy] - (c1 * (n2p - n2) - c2 * (n1p - n1));
#if PMHD_CELL_CARRY_E
      q2 = n2; q2p = n2p; q1 = n1; q1p = n1p;
#endif
      // faces: b1 at i (and ie on the rim), b2 at j (and je), b3 at k (and ke)
      if (!push || i != G.is) STC(Sout[5] + id, b1lo);
      if (i == G.ie - 1) STC(Sout[5] + id + 1, b1hi);
      STC(Sout[6] + id, b2lo);
      if (j == G.je - 1) STC(Sout[6] + id + sx, b2hi);
      STC(Sout[7] + id, b3lo);
      if (k + 1 == G.ke) STC(Sout[7] + id + sy, b3hi);
      if (push) {
        if (i > G.is && i <= G.is + G.ng) STC(PL[5] + id + mb0, b1lo);
        if (i >= G.ie - G.ng) STC(PR[5] + id - mb0, b1lo);
        if (i == G.ie - 1) {
          if (G.ie <= G.is + G.ng) STC(PL[5] + id + 1 + mb0, b1hi);
          STC(PR[5] + id + 1 - mb0, b1hi);
        }
        push_cell(6, id, b2lo);
        if (j == G.je - 1) push_cell(6, id + sx, b2hi);
        push_cell(7, id, b3lo);
        if (k + 1 == G.ke) push_cell(7, id + sy, b3hi);
      }
      // conserved update, cons_to_prim with floors, dt
      double u[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        double du = c1 * (X1[v][id + 1] - X1[v][id]) + c2 * (X2[v][id + sx] - X2[v][id]);
        if (D3) {
#if PMHD_CELL_CARRY_X3
          const double f3n = X3[v][id + sy];
          du = du + c3 * (f3n - f3[v]);
          f3[v] = f3n;
#else
          du = du + c3 * (X3[v][id + sy] - X3[v][id]);
#endif
        }
        u[v] = Sb[v][id] - du;
      }
      double bc[3], w[8];
      bc[0] = 0.5 * (b1lo + b1hi);
      bc[1] = 0.5 * (b2lo + b2hi);
      bc[2] = 0.5 * (b3lo + b3hi);
      const int fl = cons_to_prim(u, bc, ph, w, true);
      if (fl & 3)
        atomicAdd(&red[ks.stage].floor_count,
                  (unsigned long long)(((fl & 1) ? 1 : 0) + ((fl & 2) ? 1 : 0)));
      if (fl & 4) {
        const long long gi = (long long)B.c[0] * G.mb[0] + (i - G.is);
        const long long gj = (long long)B.c[1] * G.mb[1] + (j - G.js);
        const long long gk = D3 ? (long long)B.c[2] * G.mb[2] + (k - G.ks) : 0;
        atomicMin(&red[ks.stage].bad_key, (unsigned long long)((gk * G.nx[1] + gj) * G.nx[0] + gi));
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) STC(Sout[v] + id, u[v]);
      if (push) {
#pragma unroll
        for (int v = 0; v < 5; ++v) push_cell(v, id, u[v]);
      }
      if (want_dt) {
        const double d = w[0], p = w[4];
        const double cf1 = fast_speed_n(d, p, w[5], w[6], w[7], ph.gamma);
        const double cf2 = fast_speed_n(d, p, w[6], w[7], w[5], ph.gamma);
        double t = fmin(ddiv(G.dx[0], fabs(w[1]) + cf1), ddiv(G.dx[1], fabs(w[2]) + cf2));
        if (D3) {
          const double cf3 = fast_speed_n(d, p, w[7], w[5], w[6], ph.gamma);
          t = fmin(t, ddiv(G.dx[2], fabs(w[3]) + cf3));
        }
        tmin = fmin(tmin, t);
      }
      b3lo = b3hi;
    }
  }
  if (want_dt) {
    for (int o = 16; o > 0; o >>= 1) tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
    if ((tid & 31) == 0) redbuf[tid >> 5] = tmin;
    __syncthreads();
    if (tid < 32) {
      double v = (tid < CTHR / 32) ? redbuf[tid] : 1.0e300;
      for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (tid == 0) atomicMin(&red[0].dt_bits, (unsigned long long)__double_as_longlong(v));
    }
  }
}

}  // namespace

namespace {
// segment length: PMHD_EMF_SEG planes, or 4 / 1 when the mesh is too small
// to give ~2 waves of cell-update CTAs at PMHD_CELL_MINB per SM otherwise
int emf_seg(const KGeom& G, int kr0, int kr1) {
  const int cols = ((G.ie - G.is + CX - 1) / CX) * ((G.je - G.js + CY - 1) / CY) * G.nb;
  const int want = (2 * 148 * PMHD_CELL_MINB + cols - 1) / cols;  // segments per column
  const int fit = (kr1 - kr0 + want - 1) / want;                    // planes per segment
  return (fit >= PMHD_EMF_SEG) ? PMHD_EMF_SEG : (fit >= 4 ? 4 : 1);
}

template <int SEG>
void launch_emf_seg(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks, const KStage* kd,
                    DevRed* red, int want_dt, int kr0, int kr1, cudaStream_t s, int push, int all_local) {
  {
    // rim images need every neighbour on this rank; along k also the whole block
    const int rim = all_local ? (1 | ((kr0 == G.ks && kr1 == G.ke) ? 2 : 0)) : 0;
    const int r1 = rim & 1, kext = (rim & 2) ? kr1 : kr1 + 1;
    const int nseg = (kext - kr0 + SEG - 1) / SEG;
    const dim3 grid((G.ie - G.is + 1 - r1 + CX - 1) / CX, (G.je - G.js + 1 - r1 + CY - 1) / CY, nseg * G.nb);
    k_edge_emf<SEG><<<grid, CTHR, 0, s>>>(blks, G, ph, kd, kr0, kr1, rim);
  }
  {
    const int nseg = (kr1 - kr0 + SEG - 1) / SEG;
    const dim3 grid((G.ie - G.is + CX - 1) / CX, (G.je - G.js + CY - 1) / CY, nseg * G.nb);
    k_cell_update<SEG, true><<<grid, CTHR, 0, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, push);
  }
}
}  // namespace

bool update_emf_fills(const KGeom& G, int kr0, int kr1) {
  // PMHD_EMF_SMALL=1 (default): every 3D mesh, the segments shortened to
  // fill the GPU; 0: only meshes that fill it with full-length segments
  // (smaller ones keep k_update_fused)
#ifndef PMHD_EMF_SMALL
#define PMHD_EMF_SMALL 1
#endif
  if (PMHD_EMF_SMALL) return true;
  const long long ctas = (long long)((G.ie - G.is + CX - 1) / CX) * ((G.je - G.js + CY - 1) / CY) *
                         ((kr1 - kr0 + PMHD_EMF_SEG - 1) / PMHD_EMF_SEG) * G.nb;
  return ctas >= 2LL * 148 * PMHD_CELL_MINB;
}

void launch_update_emf(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks,
                       const KStage* kd, DevRed* red, int want_dt, int kr0, int kr1, cudaStream_t s, int push,
                       int all_local) {
  if (G.dim == 2) {  // one cell plane: E3, then the cell update
    const int r1 = all_local ? 1 : 0;
    const dim3 ge((G.ie - G.is + 1 - r1 + CX - 1) / CX, (G.je - G.js + 1 - r1 + CY - 1) / CY, G.nb);
    k_edge_emf2d<<<ge, CTHR, 0, s>>>(blks, G, ph, kd, r1);
    const dim3 gc((G.ie - G.is + CX - 1) / CX, (G.je - G.js + CY - 1) / CY, G.nb);
    k_cell_update<1, false><<<gc, CTHR, 0, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, push);
    return;
  }
  const int seg = emf_seg(G, kr0, kr1);
  if (seg == PMHD_EMF_SEG)
    launch_emf_seg<PMHD_EMF_SEG>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, s, push, all_local);
  else if (seg == 4)
    launch_emf_seg<4>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, s, push, all_local);
  else
    launch_emf_seg<1>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, s, push, all_local);
}

}  // namespace pmhd_gpu
