// kernels_split.cu -- first sm_100a implementation of the VL2 stage: one
// kernel per reference op (cons_to_prim, Riemann per direction, ct_emf,
// integrate + ct_update, end-of-stage cons_to_prim + dt, exchange sweeps).
// Every kernel covers all MeshBlocks of the mesh in one launch (blockIdx.z =
// block x k-plane).  It mirrors the oracle loop for loop, so it is also the
// debugging reference for the fused stage kernel (kernels_fused.cu).
#include "kernels.cuh"

namespace pmhd_gpu {

namespace {

struct Box {
  int k0, k1, j0, j1, i0, i1;
  int nk() const { return k1 - k0; }
  int nj() const { return j1 - j0; }
  int ni() const { return i1 - i0; }
};

constexpr int TX = 64, TY = 2;

dim3 grid_for(const Box& b, int nb) {
  return dim3((b.ni() + TX - 1) / TX, (b.nj() + TY - 1) / TY, b.nk() * nb);
}

#define BOX_INDEX(bx)                                                  \
  const int i = (bx).i0 + blockIdx.x * TX + threadIdx.x;               \
  const int j = (bx).j0 + blockIdx.y * TY + threadIdx.y;               \
  const int nkk = (bx).k1 - (bx).k0;                                   \
  const int b = blockIdx.z / nkk;                                      \
  const int k = (bx).k0 + (int)(blockIdx.z % nkk);                     \
  if (i >= (bx).i1 || j >= (bx).j1) return;

__device__ __forceinline__ unsigned long long dbits(double x) { return __double_as_longlong(x); }

__device__ __forceinline__ bool is_active(const KGeom& G, int k, int j, int i) {
  return k >= G.ks && k < G.ke && j >= G.js && j < G.je && i >= G.is && i < G.ie;
}

__device__ __forceinline__ unsigned long long global_key(const KGeom& G, const DevBlock& B, int k,
                                                         int j, int i) {
  const long long gi = (long long)B.c[0] * G.mb[0] + (i - G.is);
  const long long gj = (long long)B.c[1] * G.mb[1] + (j - G.js);
  const long long gk = (G.dim == 3) ? (long long)B.c[2] * G.mb[2] + (k - G.ks) : 0;
  return (unsigned long long)((gk * G.nx[1] + gj) * G.nx[0] + gi);
}

// Block-wide min of a positive double, then one atomicMin on its bits.
__device__ __forceinline__ void block_min_atomic(double v, unsigned long long* slot) {
  __shared__ double sm[32];
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = (threadIdx.y * blockDim.x + threadIdx.x) & 31;
  const int warp = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
  const int nw = (blockDim.x * blockDim.y + 31) >> 5;
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = (lane < nw) ? sm[lane] : 1.0e300;
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) atomicMin(slot, dbits(v));
  }
}

__device__ __forceinline__ void block_max_atomic(double v, unsigned long long* slot) {
  __shared__ double sm[32];
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = (threadIdx.y * blockDim.x + threadIdx.x) & 31;
  const int warp = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
  const int nw = (blockDim.x * blockDim.y + 31) >> 5;
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = (lane < nw) ? sm[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) atomicMax(slot, dbits(v));
  }
}

__device__ __forceinline__ double dt_cell(const KGeom& G, const KPhys& ph, const double* w) {
  const double d = w[0], p = w[4];
  const double c1 = fast_speed_n(d, p, w[5], w[6], w[7], ph.gamma);
  const double c2 = fast_speed_n(d, p, w[6], w[7], w[5], ph.gamma);
  double t = fmin(G.dx[0] / (fabs(w[1]) + c1), G.dx[1] / (fabs(w[2]) + c2));
  if (G.dim == 3) {
    const double c3 = fast_speed_n(d, p, w[7], w[5], w[6], ph.gamma);
    t = fmin(t, G.dx[2] / (fabs(w[3]) + c3));
  }
  return t;
}

__device__ __forceinline__ void load_bcc(double* const* S, const KGeom& G, int id, double* bc) {
  bc[0] = 0.5 * (S[5][id] + S[5][id + 1]);
  bc[1] = 0.5 * (S[6][id] + S[6][id + G.sx]);
  bc[2] = 0.5 * (S[7][id] + S[7][id + G.sy]);
}

//------------------------------------------------------------------ kernels
__global__ void __launch_bounds__(TX* TY) k_c2p_all(const DevBlock* __restrict__ blks, KGeom G,
                                                    KPhys ph, int sel, DevRed* red, Box bx, int stage) {
  BOX_INDEX(bx);
  const DevBlock& B = blks[b];
  double* const* S = B.st[sel];
  const int id = G.idx(k, j, i);
  double u[5], bc[3], w[8];
#pragma unroll
  for (int v = 0; v < 5; ++v) u[v] = S[v][id];
  load_bcc(S, G, id, bc);
  const int fl = cons_to_prim(u, bc, ph, w, false);
#pragma unroll
  for (int v = 0; v < 8; ++v) B.w[v][id] = w[v];
  if ((fl & 4) && is_active(G, k, j, i)) atomicMin(&red[stage].bad_key, global_key(G, B, k, j, i));
}

template <int DIR>
__global__ void __launch_bounds__(TX* TY) k_flux(const DevBlock* __restrict__ blks, KGeom G, KPhys ph,
                                                 int sel, int plm, double c1024, Box bx) {
  BOX_INDEX(bx);
  const DevBlock& B = blks[b];
  const int off = (DIR == 0) ? 1 : ((DIR == 1) ? G.sx : G.sy);
  // rotated variable map: (d, vn, vt1, vt2, p, bt1, bt2)
  constexpr int V0 = 0, V4 = 4;
  constexpr int V1 = (DIR == 0) ? 1 : ((DIR == 1) ? 2 : 3);
  constexpr int V2 = (DIR == 0) ? 2 : ((DIR == 1) ? 3 : 1);
  constexpr int V3 = (DIR == 0) ? 3 : ((DIR == 1) ? 1 : 2);
  constexpr int V5 = (DIR == 0) ? 6 : ((DIR == 1) ? 7 : 5);
  constexpr int V6 = (DIR == 0) ? 7 : ((DIR == 1) ? 5 : 6);
  const int vars[7] = {V0, V1, V2, V3, V4, V5, V6};
  const int id = G.idx(k, j, i);
  double wl[7], wr[7];
#pragma unroll
  for (int n = 0; n < 7; ++n) {
    const double* __restrict__ q = B.w[vars[n]];
    const double qm1 = __ldg(q + id - off), q0 = __ldg(q + id);
    if (plm) {
      const double qm2 = __ldg(q + id - 2 * off), qp1 = __ldg(q + id + off);
      wl[n] = qm1 + 0.5 * plm_slope(qm2, qm1, q0, ph.limiter);
      wr[n] = q0 - 0.5 * plm_slope(qm1, q0, qp1, ph.limiter);
    } else {
      wl[n] = qm1;
      wr[n] = q0;
    }
  }
  double out[8];
  face_solve(wl, wr, B.st[sel][5 + DIR][id], ph, c1024, out);  // (no fallback count: debug path)
  double* const* F = B.fx[DIR];
  F[0][id] = out[0];
  F[V1][id] = out[1];
  F[V2][id] = out[2];
  F[V3][id] = out[3];
  F[4][id] = out[4];
  F[5][id] = out[5];
  F[6][id] = out[6];
  F[7][id] = out[7];
}

__device__ __forceinline__ double ecc(const DevBlock& B, int comp, int id) {
  const double v1 = B.w[1][id], v2 = B.w[2][id], v3 = B.w[3][id];
  const double b1 = B.w[5][id], b2 = B.w[6][id], b3 = B.w[7][id];
  if (comp == 0) return v3 * b2 - v2 * b3;
  if (comp == 1) return v1 * b3 - v3 * b1;
  return v2 * b1 - v1 * b2;
}

__global__ void __launch_bounds__(TX* TY) k_emf(const DevBlock* __restrict__ blks, KGeom G, KPhys ph,
                                                Box bx) {
  BOX_INDEX(bx);
  const DevBlock& B = blks[b];
  const int id = G.idx(k, j, i), sx = G.sx, sy = G.sy;
  double* const* X1 = B.fx[0];
  double* const* X2 = B.fx[1];
  double* const* X3 = B.fx[2];
  const int mode = ph.emf;
  if (k < G.ke) {
    B.e[2][id] = corner_emf(mode, X1[5][id], X1[5][id - sx], X2[6][id], X2[6][id - 1], X1[7][id],
                            X1[7][id - sx], X2[7][id], X2[7][id - 1], ecc(B, 2, id), ecc(B, 2, id - 1),
                            ecc(B, 2, id - sx), ecc(B, 2, id - sx - 1));
  }
  if (G.dim == 3) {
    if (i < G.ie)
      B.e[0][id] = corner_emf(mode, X2[5][id], X2[5][id - sy], X3[6][id], X3[6][id - sx], X2[7][id],
                              X2[7][id - sy], X3[7][id], X3[7][id - sx], ecc(B, 0, id),
                              ecc(B, 0, id - sx), ecc(B, 0, id - sy), ecc(B, 0, id - sy - sx));
    if (j < G.je)
      B.e[1][id] = corner_emf(mode, X3[5][id], X3[5][id - 1], X1[6][id], X1[6][id - sy], X3[7][id],
                              X3[7][id - 1], X1[7][id], X1[7][id - sy], ecc(B, 1, id),
                              ecc(B, 1, id - sy), ecc(B, 1, id - 1), ecc(B, 1, id - sy - 1));
  } else {
    if (i < G.ie) { const double e = X2[5][id]; B.e[0][id] = e; B.e[0][id + sy] = e; }
    if (j < G.je) { const double e = X1[6][id]; B.e[1][id] = e; B.e[1][id + sy] = e; }
  }
}

__global__ void __launch_bounds__(TX* TY) k_update(const DevBlock* __restrict__ blks, KGeom G,
                                                   KStage ks, Box bx) {
  BOX_INDEX(bx);
  const DevBlock& B = blks[b];
  const int id = G.idx(k, j, i), sx = G.sx, sy = G.sy;
  double* const* base = B.st[0];
  double* const* out = B.st[ks.out_sel];
  const bool d3 = (G.dim == 3);
  const double c1 = ks.c1, c2 = ks.c2, c3 = ks.c3;
  const bool kin = k < G.ke, jin = j < G.je, iin = i < G.ie;
  if (kin && jin && iin) {
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      const double* X1 = B.fx[0][v];
      const double* X2 = B.fx[1][v];
      double du = c1 * (X1[id + 1] - X1[id]) + c2 * (X2[id + sx] - X2[id]);
      if (d3) {
        const double* X3 = B.fx[2][v];
        du = du + c3 * (X3[id + sy] - X3[id]);
      }
      out[v][id] = base[v][id] - du;
    }
  }
  const double* e1 = B.e[0];
  const double* e2 = B.e[1];
  const double* e3 = B.e[2];
  if (kin && jin) {
    if (d3) out[5][id] = base[5][id] - (c2 * (e3[id + sx] - e3[id]) - c3 * (e2[id + sy] - e2[id]));
    else out[5][id] = base[5][id] - c2 * (e3[id + sx] - e3[id]);
  }
  if (kin && iin) {
    if (d3) out[6][id] = base[6][id] - (c3 * (e1[id + sy] - e1[id]) - c1 * (e3[id + 1] - e3[id]));
    else out[6][id] = base[6][id] + c1 * (e3[id + 1] - e3[id]);
  }
  if (jin && iin) {
    const long long ie = d3 ? id : id - (long long)k * sy;  // 2D: both layers use k = 0 edges
    out[7][id] = base[7][id] - (c1 * (e2[ie + 1] - e2[ie]) - c2 * (e1[ie + sx] - e1[ie]));
  }
}

__global__ void __launch_bounds__(TX* TY) k_c2p_end(const DevBlock* __restrict__ blks, KGeom G,
                                                    KPhys ph, KStage ks, DevRed* red, int want_dt,
                                                    Box bx) {
  const int i = bx.i0 + blockIdx.x * TX + threadIdx.x;
  const int j = bx.j0 + blockIdx.y * TY + threadIdx.y;
  const int nkk = bx.k1 - bx.k0;
  const int b = blockIdx.z / nkk;
  const int k = bx.k0 + (int)(blockIdx.z % nkk);
  double tmin = 1.0e300;
  if (i < bx.i1 && j < bx.j1) {
    const DevBlock& B = blks[b];
    double* const* S = B.st[ks.out_sel];
    const int id = G.idx(k, j, i);
    double u[5], bc[3], w[8];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = S[v][id];
    load_bcc(S, G, id, bc);
    const int fl = cons_to_prim(u, bc, ph, w, true);
    if (fl & 3) {
      atomicAdd(&red[ks.stage].floor_count, (unsigned long long)(((fl & 1) ? 1 : 0) + ((fl & 2) ? 1 : 0)));
#pragma unroll
      for (int v = 0; v < 5; ++v) S[v][id] = u[v];
    }
    if (fl & 4) atomicMin(&red[ks.stage].bad_key, global_key(G, B, k, j, i));
    if (want_dt) tmin = dt_cell(G, ph, w);
  }
  if (want_dt) block_min_atomic(tmin, &red[0].dt_bits);
}

__global__ void __launch_bounds__(TX* TY) k_dt_state(const DevBlock* __restrict__ blks, KGeom G,
                                                     KPhys ph, DevRed* red, Box bx) {
  const int i = bx.i0 + blockIdx.x * TX + threadIdx.x;
  const int j = bx.j0 + blockIdx.y * TY + threadIdx.y;
  const int nkk = bx.k1 - bx.k0;
  const int b = blockIdx.z / nkk;
  const int k = bx.k0 + (int)(blockIdx.z % nkk);
  double tmin = 1.0e300;
  if (i < bx.i1 && j < bx.j1) {
    const DevBlock& B = blks[b];
    double* const* S = B.st[0];
    const int id = G.idx(k, j, i);
    double u[5], bc[3], w[8];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = S[v][id];
    load_bcc(S, G, id, bc);
    const int fl = cons_to_prim(u, bc, ph, w, false);
    if (fl & 4) atomicMin(&red[0].bad_key, global_key(G, B, k, j, i));
    tmin = dt_cell(G, ph, w);
  }
  block_min_atomic(tmin, &red[0].dt_bits);
}

__global__ void __launch_bounds__(TX* TY) k_divb(const DevBlock* __restrict__ blks, KGeom G,
                                                 DevRed* red, Box bx) {
  const int i = bx.i0 + blockIdx.x * TX + threadIdx.x;
  const int j = bx.j0 + blockIdx.y * TY + threadIdx.y;
  const int nkk = bx.k1 - bx.k0;
  const int b = blockIdx.z / nkk;
  const int k = bx.k0 + (int)(blockIdx.z % nkk);
  double m = 0.0;
  if (i < bx.i1 && j < bx.j1) {
    double* const* S = blks[b].st[0];
    const int id = G.idx(k, j, i);
    const double d = (S[5][id + 1] - S[5][id]) / G.dx[0] + (S[6][id + G.sx] - S[6][id]) / G.dx[1] +
                     (S[7][id + G.sy] - S[7][id]) / G.dx[2];
    m = fabs(d);
  }
  block_max_atomic(m, &red[0].divb_bits);
}

// One thread per (block, variable, active row): serial sum over i, so the
// total is summed in the oracle's fixed order (row sums, rows in k-j order).
__global__ void k_row_sums(const DevBlock* __restrict__ blks, KGeom G, double* rows) {
  const int nrow = (G.ke - G.ks) * (G.je - G.js);
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)G.nb * 5 * nrow) return;
  const int r = (int)(t % nrow);
  const int v = (int)((t / nrow) % 5);
  const int b = (int)(t / (5LL * nrow));
  const int k = G.ks + r / (G.je - G.js), j = G.js + r % (G.je - G.js);
  const double* q = blks[b].st[0][v];
  double s = 0.0;
  for (int i = G.is; i < G.ie; ++i) s += q[G.idx(k, j, i)];
  rows[t] = s;
}

// Exchange sweep in direction DIR (exchange_ghosts).
// Layer slot l in [0, 2 ng + 1): l < ng lower ghosts (l <= ng for the normal
// face array), the rest upper.  For x1 the layers of one row are a few
// doubles apart, so one thread copies all of them (loads first: more bytes
// in flight per thread on this latency-bound strided copy); x2 / x3 use one
// thread per (row, layer).
__device__ __forceinline__ bool exch_layer(const KGeom& G, const DevBlock& B, int DIR, int v, int l, int* q,
                                           int* qs, int* nb, int* side) {
  const int ng = G.ng, m = G.mb[DIR];
  const int e = ng + m;
  const bool normal = (v == 5 + DIR);
  if (!normal) {
    if (l < ng) { *q = l; *qs = l + m; *side = 0; }
    else if (l < 2 * ng) { *q = e + (l - ng); *qs = *q - m; *side = 1; }
    else return false;
  } else {
    if (l <= ng) { *q = l; *qs = l + m; *side = 0; }
    else { *q = e + 1 + (l - ng - 1); *qs = *q - m; *side = 1; }
  }
  *nb = B.nbr[DIR][*side];
  // remote neighbour: read over peer memory if attached, else the halo
  // unpack fills it
  return *nb >= 0 || B.rbase[DIR][*side] != nullptr;
}

// source array of the copy: the local neighbour's, or the remote one's
// (same offset from its block base)
__device__ __forceinline__ const double* exch_src(const DevBlock* blks, const DevBlock& B, int DIR, int side,
                                                  int nb, int sel, int v) {
  if (nb >= 0) return blks[nb].st[sel][v];
  const char* own = reinterpret_cast<const char*>(B.st[sel][v]);
  return reinterpret_cast<const double*>(B.rbase[DIR][side] + (own - B.base));
}

template <int DIR>
__global__ void k_exchange(const DevBlock* __restrict__ blks, KGeom G, int sel, const KStage* kd) {
  if (kd && kd->skip) return;  // graph-replayed cycle past the end of the run
  const int v = blockIdx.z % kNState;
  const int b = blockIdx.z / kNState;
  const int e1 = G.n1 + (v == 5), e2 = G.n2 + (v == 6), e3 = G.n3 + (v == 7);
  const int ta = (DIR == 2) ? e2 : e3;      // slow transverse extent
  const int tb = (DIR == 0) ? e2 : e1;      // fast transverse extent
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (long long)ta * tb) return;
  const int a = (int)(p / tb), c = (int)(p % tb);
  const DevBlock& B = blks[b];
  auto at = [&](int qq) {
    if (DIR == 0) return G.idx(a, c, qq);
    if (DIR == 1) return G.idx(a, qq, c);
    return G.idx(qq, a, c);
  };
  if (DIR == 0) {
    constexpr int MAXL = 9;  // 2 ng + 1 for ng <= 4
    double val[MAXL];
    int dst[MAXL], nbs[MAXL];
    const int nl = 2 * G.ng + 1;
#pragma unroll
    for (int l = 0; l < MAXL; ++l) {
      nbs[l] = 0;
      int q, qs, nb, side;
      if (l < nl && exch_layer(G, B, DIR, v, l, &q, &qs, &nb, &side)) {
        PMHD_CHECK_ID(G, at(qs));
        PMHD_CHECK_ID(G, at(q));
        val[l] = exch_src(blks, B, DIR, side, nb, sel, v)[at(qs)];
        dst[l] = at(q);
        nbs[l] = 1;
      }
    }
#pragma unroll
    for (int l = 0; l < MAXL; ++l)
      if (nbs[l]) B.st[sel][v][dst[l]] = val[l];
  } else {
    int q, qs, nb, side;
    if (!exch_layer(G, B, DIR, v, blockIdx.y, &q, &qs, &nb, &side)) return;
    PMHD_CHECK_ID(G, at(qs));
    PMHD_CHECK_ID(G, at(q));
    B.st[sel][v][at(q)] = exch_src(blks, B, DIR, side, nb, sel, v)[at(qs)];
  }
}

}  // namespace

//------------------------------------------------------------------ launchers
static Box all_cells(const KGeom& G) { return Box{0, G.n3, 0, G.n2, 0, G.n1}; }
static Box active(const KGeom& G) { return Box{G.ks, G.ke, G.js, G.je, G.is, G.ie}; }
static dim3 tb() { return dim3(TX, TY, 1); }

void launch_c2p_all(const DevBlock* blks, const KGeom& G, const KPhys& ph, int sel, DevRed* red,
                    int stage, cudaStream_t s) {
  const Box bx = all_cells(G);
  k_c2p_all<<<grid_for(bx, G.nb), tb(), 0, s>>>(blks, G, ph, sel, red, bx, stage);
}

void launch_flux(const DevBlock* blks, const KGeom& G, const KPhys& ph, int dir, int sel, int plm,
                 double c1024, cudaStream_t s) {
  const int d3 = (G.dim == 3) ? 1 : 0;
  Box bx;
  if (dir == 0) bx = Box{G.ks - d3, G.ke + d3, G.js - 1, G.je + 1, G.is, G.ie + 1};
  else if (dir == 1) bx = Box{G.ks - d3, G.ke + d3, G.js, G.je + 1, G.is - 1, G.ie + 1};
  else bx = Box{G.ks, G.ke + 1, G.js - 1, G.je + 1, G.is - 1, G.ie + 1};
  const dim3 g = grid_for(bx, G.nb);
  if (dir == 0) k_flux<0><<<g, tb(), 0, s>>>(blks, G, ph, sel, plm, c1024, bx);
  else if (dir == 1) k_flux<1><<<g, tb(), 0, s>>>(blks, G, ph, sel, plm, c1024, bx);
  else k_flux<2><<<g, tb(), 0, s>>>(blks, G, ph, sel, plm, c1024, bx);
}

void launch_emf(const DevBlock* blks, const KGeom& G, const KPhys& ph, cudaStream_t s) {
  const int d3 = (G.dim == 3) ? 1 : 0;
  const Box bx{G.ks, G.ke + d3, G.js, G.je + 1, G.is, G.ie + 1};
  k_emf<<<grid_for(bx, G.nb), tb(), 0, s>>>(blks, G, ph, bx);
}

void launch_update(const DevBlock* blks, const KGeom& G, const KStage& ks, cudaStream_t s) {
  const Box bx{G.ks, (G.dim == 3) ? G.ke + 1 : 2, G.js, G.je + 1, G.is, G.ie + 1};
  k_update<<<grid_for(bx, G.nb), tb(), 0, s>>>(blks, G, ks, bx);
}

void launch_c2p_end(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks,
                    DevRed* red, int want_dt, cudaStream_t s) {
  const Box bx = active(G);
  k_c2p_end<<<grid_for(bx, G.nb), tb(), 0, s>>>(blks, G, ph, ks, red, want_dt, bx);
}

void launch_exchange(const DevBlock* blks, const KGeom& G, int sel, cudaStream_t s, const KStage* kd) {
  for (int dir = 0; dir < G.dim; ++dir) launch_exchange_dir(blks, G, sel, dir, s, kd);
}

void launch_exchange_dir(const DevBlock* blks, const KGeom& G, int sel, int dir, cudaStream_t s,
                         const KStage* kd) {
  {
    long long plane;
    if (dir == 0) plane = (long long)(G.n3 + 1) * (G.n2 + 1);
    else if (dir == 1) plane = (long long)(G.n3 + 1) * (G.n1 + 1);
    else plane = (long long)(G.n2 + 1) * (G.n1 + 1);
    // (x1: one thread per row does every layer; ng <= 4 is validated)
    const dim3 g((unsigned)((plane + 255) / 256), dir == 0 ? 1 : 2 * G.ng + 1, G.nb * kNState);
    if (dir == 0) k_exchange<0><<<g, 256, 0, s>>>(blks, G, sel, kd);
    else if (dir == 1) k_exchange<1><<<g, 256, 0, s>>>(blks, G, sel, kd);
    else k_exchange<2><<<g, 256, 0, s>>>(blks, G, sel, kd);
  }
}

void launch_dt_from_state(const DevBlock* blks, const KGeom& G, const KPhys& ph, DevRed* red,
                          cudaStream_t s) {
  const Box bx = active(G);
  k_dt_state<<<grid_for(bx, G.nb), tb(), 0, s>>>(blks, G, ph, red, bx);
}

void launch_divb(const DevBlock* blks, const KGeom& G, DevRed* red, cudaStream_t s) {
  const Box bx = active(G);
  k_divb<<<grid_for(bx, G.nb), tb(), 0, s>>>(blks, G, red, bx);
}

void launch_row_sums(const DevBlock* blks, const KGeom& G, double* rows, cudaStream_t s) {
  const long long n = (long long)G.nb * 5 * (G.ke - G.ks) * (G.je - G.js);
  k_row_sums<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(blks, G, rows);
}

}  // namespace pmhd_gpu
