// kernels_flux.cu -- fused (cons_to_prim + reconstruction + Riemann) face-flux
// kernel, one launch per direction per stage over all MeshBlocks.
//
// Replaces the reference ops plm_reconstruct + riemann (the
// "reconstruct" and "riemann" regions of SPEC.md:527) and the stage-input
// cons_to_prim for the cells each tile touches.
//
// Tiling: a CTA of 128 threads owns 32 x 8 faces: 32 consecutive faces along
// i (coalesced HBM rows) times 8 positions along the second tile axis (j for
// x1/x2 faces, k for x3 faces) in one plane (x1/x2) or one row (x3).  The
// stencil cells of the tile (36 x 8 for x1, 32 x 11 for x2/x3) are loaded once
// with coalesced loads, converted to primitives (7 rotated variables) and kept
// in shared memory; each thread then solves 2 faces reading its stencil from
// shared memory, so no warp waits on HBM during the Riemann solve.  Several
// CTAs per SM overlap one tile's load phase with other tiles' solves.
#include "kernels.cuh"

namespace pmhd_gpu {

namespace {

constexpr int FX = 32;  // faces along i per tile
constexpr int FS = 8;   // faces along the second tile axis
constexpr int NTHR = 128;
#ifndef PMHD_FLUX_MINB
#define PMHD_FLUX_MINB 4
#endif

template <int DIR>
struct TileShape {
  static constexpr int NCOL = (DIR == 0) ? FX + 4 : FX;  // cells along i
  static constexpr int NROW = (DIR == 0) ? FS : FS + 3;  // cells along the 2nd axis
  static constexpr int NCELL = NCOL * NROW;
};

// Lab index of the 7 rotated variables (d, vn, vt1, vt2, p, bt1, bt2).
template <int DIR>
__device__ __forceinline__ int rot_var(int n) {
  constexpr int V[3][7] = {{0, 1, 2, 3, 4, 6, 7}, {0, 2, 3, 1, 4, 7, 5}, {0, 3, 1, 2, 4, 5, 6}};
  return V[DIR][n];
}

template <int DIR>
__global__ void __launch_bounds__(NTHR, PMHD_FLUX_MINB)
k_flux_fused(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, int sel, int plm, double c1024, int stage,
             DevRed* red, int f_i0, int f_i1, int f_s0, int f_s1, int f_t0, int f_t1) {
  using TS = TileShape<DIR>;
  __shared__ double sw[7][TS::NCELL];

  const int nt = f_t1 - f_t0;
  const int b = blockIdx.z / nt;
  const int t3 = f_t0 + (int)(blockIdx.z % nt);   // k for x1/x2, j for x3
  const int fi0 = f_i0 + blockIdx.x * FX;          // first face along i
  const int fs0 = f_s0 + blockIdx.y * FS;          // first face along the 2nd axis
  const DevBlock& B = blks[b];
  double* const* S = B.st[sel];

  // ---- phase 1: load + cons_to_prim of the stencil cells into smem --------
  for (int c = threadIdx.x; c < TS::NCELL; c += NTHR) {
    const int col = c % TS::NCOL, row = c / TS::NCOL;
    int i, j, k;
    if (DIR == 0) { i = fi0 - 2 + col; j = fs0 + row; k = t3; }
    else if (DIR == 1) { i = fi0 + col; j = fs0 - 2 + row; k = t3; }
    else { i = fi0 + col; k = fs0 - 2 + row; j = t3; }
    if (i < 0 || i >= G.n1 || j < 0 || j >= G.n2 || k < 0 || k >= G.n3) continue;
    const long long id = G.idx(k, j, i);
    double u[5], bc[3], w[8];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = __ldg(S[v] + id);
    bc[0] = 0.5 * (__ldg(S[5] + id) + __ldg(S[5] + id + 1));
    bc[1] = 0.5 * (__ldg(S[6] + id) + __ldg(S[6] + id + G.sx));
    bc[2] = 0.5 * (__ldg(S[7] + id) + __ldg(S[7] + id + G.sy));
    const int fl = cons_to_prim(u, bc, ph, w, false);
    if ((fl & 4) && k >= G.ks && k < G.ke && j >= G.js && j < G.je && i >= G.is && i < G.ie) {
      const long long gi = (long long)B.c[0] * G.mb[0] + (i - G.is);
      const long long gj = (long long)B.c[1] * G.mb[1] + (j - G.js);
      const long long gk = (G.dim == 3) ? (long long)B.c[2] * G.mb[2] + (k - G.ks) : 0;
      atomicMin(&red[stage].bad_key, (unsigned long long)((gk * G.nx[1] + gj) * G.nx[0] + gi));
    }
#pragma unroll
    for (int n = 0; n < 7; ++n) sw[n][c] = w[rot_var<DIR>(n)];
  }
  __syncthreads();

  // ---- phase 2: two faces per thread ---------------------------------------
  const int fc = threadIdx.x % FX;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int fr = threadIdx.x / FX + 4 * h;
    const int fi = fi0 + fc, fs = fs0 + fr;
    if (fi >= f_i1 || fs >= f_s1) continue;
    // stencil cell index of (cell on the low side - 1) ... (high side + 1)
    int c0, dc;
    if (DIR == 0) { c0 = fr * TS::NCOL + fc; dc = 1; }
    else { c0 = fr * TS::NCOL + fc; dc = TS::NCOL; }
    double wl[7], wr[7];
#pragma unroll
    for (int n = 0; n < 7; ++n) {
      const double qm2 = sw[n][c0], qm1 = sw[n][c0 + dc];
      const double q0 = sw[n][c0 + 2 * dc], qp1 = sw[n][c0 + 3 * dc];
      if (plm) {
        wl[n] = qm1 + 0.5 * plm_slope(qm2, qm1, q0, ph.limiter);
        wr[n] = q0 - 0.5 * plm_slope(qm1, q0, qp1, ph.limiter);
      } else {
        wl[n] = qm1;
        wr[n] = q0;
      }
    }
    int i, j, k;
    if (DIR == 0) { i = fi; j = fs; k = t3; }
    else if (DIR == 1) { i = fi; j = fs; k = t3; }
    else { i = fi; k = fs; j = t3; }
    const long long id = G.idx(k, j, i);
    double out[8];
    face_solve(wl, wr, __ldg(S[5 + DIR] + id), ph, c1024, out);
    double* const* F = B.fx[DIR];
    F[0][id] = out[0];
    F[rot_var<DIR>(1)][id] = out[1];
    F[rot_var<DIR>(2)][id] = out[2];
    F[rot_var<DIR>(3)][id] = out[3];
    F[4][id] = out[4];
    F[5][id] = out[5];
    F[6][id] = out[6];
    F[7][id] = out[7];
  }
}

}  // namespace

void launch_flux_fused(const DevBlock* blks, const KGeom& G, const KPhys& ph, int dir, int sel,
                       int plm, double c1024, int stage, DevRed* red, cudaStream_t s) {
  const int d3 = (G.dim == 3) ? 1 : 0;
  // face ranges of the oracle: [lo, hi) per axis
  int i0, i1, j0, j1, k0, k1;
  if (dir == 0) { k0 = G.ks - d3; k1 = G.ke + d3; j0 = G.js - 1; j1 = G.je + 1; i0 = G.is; i1 = G.ie + 1; }
  else if (dir == 1) { k0 = G.ks - d3; k1 = G.ke + d3; j0 = G.js; j1 = G.je + 1; i0 = G.is - 1; i1 = G.ie + 1; }
  else { k0 = G.ks; k1 = G.ke + 1; j0 = G.js - 1; j1 = G.je + 1; i0 = G.is - 1; i1 = G.ie + 1; }
  const int ns0 = (dir == 2) ? k0 : j0, ns1 = (dir == 2) ? k1 : j1;
  const int nt0 = (dir == 2) ? j0 : k0, nt1 = (dir == 2) ? j1 : k1;
  const dim3 grid((i1 - i0 + FX - 1) / FX, (ns1 - ns0 + FS - 1) / FS, (nt1 - nt0) * G.nb);
  if (dir == 0)
    k_flux_fused<0><<<grid, NTHR, 0, s>>>(blks, G, ph, sel, plm, c1024, stage, red, i0, i1, ns0, ns1, nt0, nt1);
  else if (dir == 1)
    k_flux_fused<1><<<grid, NTHR, 0, s>>>(blks, G, ph, sel, plm, c1024, stage, red, i0, i1, ns0, ns1, nt0, nt1);
  else
    k_flux_fused<2><<<grid, NTHR, 0, s>>>(blks, G, ph, sel, plm, c1024, stage, red, i0, i1, ns0, ns1, nt0, nt1);
}

}  // namespace pmhd_gpu
