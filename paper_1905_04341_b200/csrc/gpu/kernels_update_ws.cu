// kernels_update_ws.cu -- the fused end of a VL2 stage for 3D meshes as a
// warp-specialised kernel (two roles in one CTA, named barriers).
//
// Same reference ops, expressions and operand order as k_update_fused
// (kernels_update.cu), so the same bits: corner EMFs (ct_emf,
// SPEC.md:191-199), constrained-transport face update (ct_update_face_b,
// SPEC.md:200-208), conserved update ("integrate"),
// face_to_center_b + end-of-stage cons_to_prim with floors / error detection
// (SPEC.md:132-140, :236-239), the compute_dt partial min.
//
// Why.  k_update_fused runs its four phases (E ring, corner EMFs, CT faces,
// conserved update) one after another behind CTA barriers: the 35 loads of
// the conserved update of plane k start only once plane k's faces are done,
// although nothing in them depends on the faces.  Here a CTA of 512 threads
// owns a 32 x 8 column tile and splits into two roles that run concurrently:
//   E role (warps 0-7):  cell-centred E ring, corner EMFs, CT faces (b1, b2 at
//                        plane k, b3 at k+1) and their stores;
//   H role (warps 8-15): the hydro fluxes and u^n of its cell -> u at plane k
//                        (no dependence on the E role), then, once the faces of
//                        plane k are in shared memory, face_to_center_b,
//                        cons_to_prim, floors, stores, dt.
// Hand-over by named barriers (bar.sync / bar.arrive; id 0 stays
// __syncthreads): id 1 synchronises the E role alone, id 2 "faces of plane k
// ready" (E arrives, H waits), id 3 "faces of plane k consumed" (H arrives, E
// waits before it overwrites them two planes later: the face buffers are
// double-buffered by plane parity, so E runs up to one plane ahead of H).
#include <atomic>

#include "kernels.cuh"

namespace pmhd_gpu {

namespace {

constexpr int WX = 32, WY = 8, WC = WX * WY, WT = 2 * WC;  // cells, threads
constexpr int WEX = WX + 2, WEY = WY + 2;                 // E box (cells i0-1 .. i0+32, j0-1 .. j0+8)

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

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

struct WsSmem {
  double ecbuf[3][2][WEY][WEX];   // cell-centred E ring, slot by plane parity
  double e3s[WY + 1][WX + 1];     // E3 at (k, j-1/2, i-1/2)
  double e1s[2][WY + 1][WX];      // E1 at k -/+ 1/2, slot by parity
  double e2s[2][WY][WX + 1];      // E2 at k -/+ 1/2
  double b1s[2][WY][WX + 1];      // new b1 at plane k, slot by plane parity
  double b2s[2][WY + 1][WX];      // new b2 at plane k
  double b3s[2][WY][WX];          // new b3 at faces k / k+1, slot by face parity
  double redbuf[WT / 32];
  long long tph[3];
};

template <int SEG, int MODE>
__global__ void __launch_bounds__(WT, 2)
k_update_ws(const DevBlock* __restrict__ blks, KGeom G, KPhys ph, KStage ks_arg, const KStage* __restrict__ kd,
            DevRed* red, int want_dt, int kr0, int kr1, int push) {
  constexpr bool PROF = (MODE == 1);
  if (MODE == 2 && kd->skip) return;
  const KStage ks = (MODE == 2) ? *kd : ks_arg;
  extern __shared__ __align__(16) unsigned char ws_smem[];
  WsSmem& SM = *reinterpret_cast<WsSmem*>(ws_smem);
  const int nseg = (kr1 - kr0 + SEG - 1) / SEG;
  const int b = blockIdx.z / nseg;
  const int kb = kr0 + (int)(blockIdx.z % nseg) * SEG;
  const int kend = min(kb + SEG, kr1);
  const int i0 = G.is + blockIdx.x * WX, j0 = G.js + blockIdx.y * WY;
  const int nx = min(WX, G.ie - i0), ny = min(WY, G.je - j0);
  const DevBlock& B = blks[b];
  double* const* Sb = B.st[0];
  double* const* Sout = B.st[ks.out_sel];
  const int sx = G.sx, sy = G.sy;
  const int mode = ph.emf;
  const double c1 = ks.c1, c2 = ks.c2, c3 = ks.c3;
  const bool erole = threadIdx.x < WC;
  const int rt = erole ? threadIdx.x : threadIdx.x - WC;  // thread index within the role
  if (PROF && threadIdx.x == 0) { SM.tph[0] = clock64(); SM.tph[1] = SM.tph[2] = 0; }
  double* const* PL = push ? blks[B.nbr[0][0]].st[ks.out_sel] : nullptr;
  double* const* PR = push ? blks[B.nbr[0][1]].st[ks.out_sel] : nullptr;
  auto push_cell = [&](int v, int i, int id, double val) {
    if (i < G.is + G.ng) { PMHD_CHECK_ID(G, id + G.mb[0]); ST(PL[v] + id + G.mb[0], val); }
    if (i >= G.ie - G.ng) { PMHD_CHECK_ID(G, id - G.mb[0]); ST(PR[v] + id - G.mb[0], val); }
  };
  double tmin = 1.0e300;

  if (erole) {
    // ====================== E role: EMFs and CT faces ==========================
    double* const* X1 = B.fx[0];
    double* const* X2 = B.fx[1];
    double* const* X3 = B.fx[2];
    auto ec = [&](int c, int sl) { return SM.ecbuf[c][sl]; };
    auto load_ec = [&](int kk) {
      const int sl = kk & 1;
      for (int q = rt; q < WEY * WEX; q += WC) {
        const int c = q % WEX, r = q / WEX;
        if (c > nx + 1 || r > ny + 1) continue;
        const int id = G.idx(kk, j0 - 1 + r, i0 - 1 + c);
        PMHD_CHECK_ID(G, id);
        ec(0, sl)[r][c] = __ldg(B.ec[0] + id);
        ec(1, sl)[r][c] = __ldg(B.ec[1] + id);
        ec(2, sl)[r][c] = __ldg(B.ec[2] + id);
      }
    };
    // E1 / E2 on the edge plane kk - 1/2 into slot h (k_update_fused's edge_emfs)
    auto edge_emfs = [&](int kk, int h) {
      const int pa = kk & 1, pm = (kk - 1) & 1;
      for (int q = rt; q < (WY + 1) * WX; q += WC) {
        const int c = q % WX, r = q / WX;
        if (c >= nx || r > ny) continue;
        const int id = G.idx(kk, j0 + r, i0 + c);
        PMHD_CHECK_ID(G, id - G.sy);
        SM.e1s[h][r][c] = corner_emf(mode, X2[5][id], X2[5][id - sy], X3[6][id], X3[6][id - sx], X2[7][id],
                                     X2[7][id - sy], X3[7][id], X3[7][id - sx], ec(0, pa)[r + 1][c + 1],
                                     ec(0, pa)[r][c + 1], ec(0, pm)[r + 1][c + 1], ec(0, pm)[r][c + 1]);
      }
      for (int q = rt; q < WY * (WX + 1); q += WC) {
        const int c = q % (WX + 1), r = q / (WX + 1);
        if (c > nx || r >= ny) continue;
        const int id = G.idx(kk, j0 + r, i0 + c);
        SM.e2s[h][r][c] = corner_emf(mode, X3[5][id], X3[5][id - 1], X1[6][id], X1[6][id - sy], X3[7][id],
                                     X3[7][id - 1], X1[7][id], X1[7][id - sy], ec(1, pa)[r + 1][c + 1],
                                     ec(1, pm)[r + 1][c + 1], ec(1, pa)[r + 1][c], ec(1, pm)[r + 1][c]);
      }
    };
    // new b3 on face plane kk from the edge EMFs in slot h
    auto face_b3 = [&](int kk, int h) {
      for (int q = rt; q < WY * WX; q += WC) {
        const int c = q % WX, r = q / WX;
        if (c >= nx || r >= ny) continue;
        const int id = G.idx(kk, j0 + r, i0 + c);
        PMHD_CHECK_ID(G, id);
        SM.b3s[h][r][c] = Sb[7][id] - (c1 * (SM.e2s[h][r][c + 1] - SM.e2s[h][r][c]) -
                                       c2 * (SM.e1s[h][r + 1][c] - SM.e1s[h][r][c]));
      }
    };
    // ---- prologue: Ec planes kb-1, kb, the edge EMFs at kb - 1/2, b3 at kb ---
    load_ec(kb - 1);
    load_ec(kb);
    named_sync(1, WC);
    edge_emfs(kb, kb & 1);
    named_sync(1, WC);
    face_b3(kb, kb & 1);
    for (int k = kb; k < kend; ++k) {
      const int lo = k & 1, hi = lo ^ 1;  // slots of k - 1/2 and k + 1/2 (and of planes k-1 / k)
      if (PROF && rt == 0 && k > kb) { const long long t = clock64(); SM.tph[2] += t - SM.tph[0]; SM.tph[0] = t; }
      load_ec(k + 1);  // into the slot of plane k-1, last read by the EMFs of step k-1
      named_sync(1, WC);
      // ---- E3 at plane k, E1 / E2 at k + 1/2 -----------------------------------
      for (int q = rt; q < (WY + 1) * (WX + 1); q += WC) {
        const int c = q % (WX + 1), r = q / (WX + 1);
        if (c > nx || r > ny) continue;
        const int id = G.idx(k, j0 + r, i0 + c);
        PMHD_CHECK_ID(G, id - G.sx);
        const int ec_c = c + 1, ec_r = r + 1;
        SM.e3s[r][c] = corner_emf(mode, X1[5][id], X1[5][id - sx], X2[6][id], X2[6][id - 1], X1[7][id],
                                  X1[7][id - sx], X2[7][id], X2[7][id - 1], ec(2, lo)[ec_r][ec_c],
                                  ec(2, lo)[ec_r][ec_c - 1], ec(2, lo)[ec_r - 1][ec_c],
                                  ec(2, lo)[ec_r - 1][ec_c - 1]);
      }
      edge_emfs(k + 1, hi);
      named_sync(1, WC);
      if (PROF && rt == 0) { const long long t = clock64(); SM.tph[1] += t - SM.tph[0]; SM.tph[0] = t; }
      // the face buffers of plane k's parity were last read by the H role at
      // step k-2; b3 slot hi (face k+1) at step k-1: wait for its hand-back
      if (k > kb) named_sync(3, WT);
      // ---- constrained-transport faces of plane k (b3 at k+1) -------------------
      const int pb = k & 1;
      for (int q = rt; q < WY * (WX + 1); q += WC) {  // b1f, faces i0 .. i0+nx
        const int c = q % (WX + 1), r = q / (WX + 1);
        if (c > nx || r >= ny) continue;
        const int id = G.idx(k, j0 + r, i0 + c);
        const double v =
            Sb[5][id] - (c2 * (SM.e3s[r + 1][c] - SM.e3s[r][c]) - c3 * (SM.e2s[hi][r][c] - SM.e2s[lo][r][c]));
        SM.b1s[pb][r][c] = v;
        if (c < nx || i0 + c == G.ie) {
          const int i = i0 + c;
          if (!push || i != G.is) ST(Sout[5] + id, v);
          if (push) {
            if (i > G.is && i <= G.is + G.ng) { PMHD_CHECK_ID(G, id + G.mb[0]); ST(PL[5] + id + G.mb[0], v); }
            if (i >= G.ie - G.ng) { PMHD_CHECK_ID(G, id - G.mb[0]); ST(PR[5] + id - G.mb[0], v); }
          }
        }
      }
      for (int q = rt; q < (WY + 1) * WX; q += WC) {  // b2f, faces j0 .. j0+ny
        const int c = q % WX, r = q / WX;
        if (c >= nx || r > ny) continue;
        const int id = G.idx(k, j0 + r, i0 + c);
        const double v =
            Sb[6][id] - (c3 * (SM.e1s[hi][r][c] - SM.e1s[lo][r][c]) - c1 * (SM.e3s[r][c + 1] - SM.e3s[r][c]));
        SM.b2s[pb][r][c] = v;
        if (r < ny || j0 + r == G.je) {
          ST(Sout[6] + id, v);
          if (push) push_cell(6, i0 + c, id, v);
        }
      }
      face_b3(k + 1, hi);  // b3 at face k + 1 (face k carried)
      {
        const int c = rt % WX, r = rt / WX;
        if (c < nx && r < ny) {
          const int id = G.idx(k, j0 + r, i0 + c);
          ST(Sout[7] + id, SM.b3s[lo][r][c]);
          if (k + 1 == G.ke) ST(Sout[7] + id + sy, SM.b3s[hi][r][c]);
          if (push) {
            push_cell(7, i0 + c, id, SM.b3s[lo][r][c]);
            if (k + 1 == G.ke) push_cell(7, i0 + c, id + sy, SM.b3s[hi][r][c]);
          }
        }
      }
      named_arrive(2, WT);  // faces of plane k ready for the H role
    }
    named_sync(3, WT);  // the H role's hand-back of the last plane
  } else {
    // ====================== H role: conserved update ===========================
    double* const* X1 = B.fx[0];
    double* const* X2 = B.fx[1];
    double* const* X3 = B.fx[2];
    const int c = rt % WX, r = rt / WX;
    const bool own = c < nx && r < ny;
    const int i = i0 + c, j = j0 + r;
    for (int k = kb; k < kend; ++k) {
      const int lo = k & 1, hi = lo ^ 1, pb = k & 1;
      double u[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      const int id = G.idx(k, j, i);
      if (own) {
        PMHD_CHECK_ID(G, id + G.sy);
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          double du = c1 * (X1[v][id + 1] - X1[v][id]) + c2 * (X2[v][id + sx] - X2[v][id]);
          du = du + c3 * (X3[v][id + sy] - X3[v][id]);
          u[v] = Sb[v][id] - du;
        }
      }
      named_sync(2, WT);  // the E role's faces of plane k
      double bc[3], w[8];
      if (own) {
        bc[0] = 0.5 * (SM.b1s[pb][r][c] + SM.b1s[pb][r][c + 1]);
        bc[1] = 0.5 * (SM.b2s[pb][r][c] + SM.b2s[pb][r + 1][c]);
        bc[2] = 0.5 * (SM.b3s[lo][r][c] + SM.b3s[hi][r][c]);
      }
      named_arrive(3, WT);  // plane k's faces consumed
      if (own) {
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
          const double d = w[0], p = w[4];
          const double cf1 = fast_speed_n(d, p, w[5], w[6], w[7], ph.gamma);
          const double cf2 = fast_speed_n(d, p, w[6], w[7], w[5], ph.gamma);
          double t = fmin(ddiv(G.dx[0], fabs(w[1]) + cf1), ddiv(G.dx[1], fabs(w[2]) + cf2));
          const double cf3 = fast_speed_n(d, p, w[7], w[5], w[6], ph.gamma);
          t = fmin(t, ddiv(G.dx[2], fabs(w[3]) + cf3));
          tmin = fmin(tmin, t);
        }
      }
    }
  }
  if (PROF) {
    __syncthreads();
    if (threadIdx.x == 0) {
      SM.tph[2] += clock64() - SM.tph[0];
      atomicAdd(&red[ks.stage].phase[3], (unsigned long long)SM.tph[1]);
      atomicAdd(&red[ks.stage].phase[4], (unsigned long long)SM.tph[2]);
    }
  }
  if (want_dt) {
    for (int o = 16; o > 0; o >>= 1) tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
    if ((threadIdx.x & 31) == 0) SM.redbuf[threadIdx.x >> 5] = tmin;
    __syncthreads();
    if (threadIdx.x < 32) {
      double v = (threadIdx.x < WT / 32) ? SM.redbuf[threadIdx.x] : 1.0e300;
      for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (threadIdx.x == 0) atomicMin(&red[0].dt_bits, (unsigned long long)__double_as_longlong(v));
    }
  }
}

}  // namespace

void launch_update_ws(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks, const KStage* kd,
                      DevRed* red, int want_dt, int kr0, int kr1, cudaStream_t s, int push) {
  // two CTAs per SM; segments of 16 planes, or 4 / 1 on small meshes (as k_update_fused)
  const int tiles = ((G.ie - G.is + WX - 1) / WX) * ((G.je - G.js + WY - 1) / WY) * G.nb;
  const int nk = kr1 - kr0;
  const int want = (2 * 148 * 2 + tiles - 1) / tiles;
  const int fit = (nk + want - 1) / want;
  const int seg = (fit >= 16) ? 16 : (fit >= 4 ? 4 : 1);
  const int nseg = (nk + seg - 1) / seg;
  const dim3 grid((G.ie - G.is + WX - 1) / WX, (G.je - G.js + WY - 1) / WY, nseg * G.nb);
  constexpr int smem = (int)sizeof(WsSmem);
#define PMHD_WS_LAUNCH(SG)                                                                                \
  do {                                                                                                    \
    static std::atomic<unsigned long long> attr_devs{0};                                                  \
    int dev = 0;                                                                                          \
    cudaGetDevice(&dev);                                                                                  \
    if (!(attr_devs.load() & (1ULL << (dev & 63)))) {                                                     \
      cudaFuncSetAttribute(k_update_ws<SG, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);        \
      cudaFuncSetAttribute(k_update_ws<SG, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);        \
      cudaFuncSetAttribute(k_update_ws<SG, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);        \
      attr_devs.fetch_or(1ULL << (dev & 63));                                                             \
    }                                                                                                     \
    if (kd) k_update_ws<SG, 2><<<grid, WT, smem, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, push); \
    else if (ph.prof) k_update_ws<SG, 1><<<grid, WT, smem, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, push); \
    else k_update_ws<SG, 0><<<grid, WT, smem, s>>>(blks, G, ph, ks, kd, red, want_dt, kr0, kr1, push); \
  } while (0)
  if (seg == 16) PMHD_WS_LAUNCH(16);
  else if (seg == 4) PMHD_WS_LAUNCH(4);
  else PMHD_WS_LAUNCH(1);
#undef PMHD_WS_LAUNCH
}

}  // namespace pmhd_gpu
