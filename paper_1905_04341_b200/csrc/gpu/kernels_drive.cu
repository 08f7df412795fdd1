// kernels_drive.cu -- turbulence driving (the "driven" phase
// of BASELINE config 5): an impulsive solenoidal velocity kick every
// turb_every cycles (definition in include/pmhd_host.h, oracle restatement
// in oracle/pmhd_oracle.hpp drive_*).  The global sums it needs are formed
// in a fixed order -- each (k, j) row summed over i, each k plane over its
// rows in j order, each block over its planes in k order, blocks combined on
// the host in gid order -- so one process, several ranks and the CPU oracle
// agree bit for bit.  Runs once per driving event, not on the timed VL2 path.
#include "kernels.cuh"

namespace pmhd_gpu {

namespace {

__device__ __forceinline__ int gidx(const KGeom& G, const DevBlock& B, int a, int l) {
  // global cell index along axis a of local index l
  const int s = (a == 0) ? G.is : (a == 1 ? G.js : G.ks);
  return B.c[a] * G.mb[a] + (l - s);
}

// dv = sum_m c_m cos(k.x) + s_m sin(k.x) on every active cell -> B.fx[0][0..2].
// One thread per (block, k-run, j, i): the x-y phase product of each mode is
// formed once and reused for the DV_KC cells of the k run; every cell still
// adds its modes in m order with the oracle's expressions.
constexpr int DV_KC = 8;

__global__ void __launch_bounds__(128) k_drive_dv(const DevBlock* __restrict__ blks, KGeom G, DriveTabs T) {
  const int ni = G.ie - G.is, nj = G.je - G.js, nk = G.ke - G.ks;
  const int nkr = (nk + DV_KC - 1) / DV_KC;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)G.nb * nkr * nj * ni) return;
  const int i = G.is + (int)(t % ni);
  const int j = G.js + (int)((t / ni) % nj);
  const int kr = (int)((t / ((long long)ni * nj)) % nkr);
  const int b = (int)(t / ((long long)ni * nj * nkr));
  const DevBlock& B = blks[b];
  const int k0 = G.ks + kr * DV_KC;
  const int kn = min(DV_KC, G.ke - k0);
  const int gi = gidx(G, B, 0, i), gj = gidx(G, B, 1, j);
  const int gk0 = (G.dim == 3) ? gidx(G, B, 2, k0) : 0;
  double dv[DV_KC][3];
#pragma unroll
  for (int c = 0; c < DV_KC; ++c) dv[c][0] = dv[c][1] = dv[c][2] = 0.0;
  for (int m = 0; m < T.n; ++m) {
    const int qx = (T.k[m][0] + 2) * G.nx[0] + gi;
    const int qy = (T.k[m][1] + 2) * G.nx[1] + gj;
    const double axr = T.ct[0][qx], axi = T.st[0][qx];
    const double ayr = T.ct[1][qy], ayi = T.st[1][qy];
    const double zr = axr * ayr - axi * ayi, zi = axr * ayi + axi * ayr;
    const double c0 = T.c[m][0], c1 = T.c[m][1], c2 = T.c[m][2];
    const double s0 = T.s[m][0], s1 = T.s[m][1], s2 = T.s[m][2];
    const double* czt = T.ct[2] + (T.k[m][2] + 2) * G.nx[2] + gk0;
    const double* szt = T.st[2] + (T.k[m][2] + 2) * G.nx[2] + gk0;
#pragma unroll
    for (int c = 0; c < DV_KC; ++c) {
      if (c < kn) {
        const double azr = czt[c], azi = szt[c];
        const double cr = zr * azr - zi * azi, ci = zr * azi + zi * azr;
        dv[c][0] = dv[c][0] + (c0 * cr + s0 * ci);
        dv[c][1] = dv[c][1] + (c1 * cr + s1 * ci);
        dv[c][2] = dv[c][2] + (c2 * cr + s2 * ci);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < DV_KC; ++c) {
    if (c < kn) {
      const int id = G.idx(k0 + c, j, i);
      B.fx[0][0][id] = dv[c][0];
      B.fx[0][1][id] = dv[c][1];
      B.fx[0][2][id] = dv[c][2];
    }
  }
}

// Per (block, k, j) row, summed over i in order.  mode 0: (rho, rho dv);
// mode 1: (1/2 rho |dv'|^2, m.dv') with dv' = dv - mean.  A CTA owns 32 rows
// and walks them in chunks of 32 cells: all 8 warps read the chunk coalesced
// and form each cell's terms; then warp q adds term q of its lane's row
// across the chunk in i order, so every row sum keeps the sequential order.
constexpr int RS_ROWS = 32;

__global__ void __launch_bounds__(256) k_drive_rows(const DevBlock* __restrict__ blks, KGeom G, int mode,
                                                    double m0, double m1, double m2, double* rows) {
  __shared__ double term[4][RS_ROWS][33];
  const int ni = G.ie - G.is, nj = G.je - G.js, nk = G.ke - G.ks;
  const int nr = G.nb * nk * nj;
  const int r0 = blockIdx.x * RS_ROWS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nterm = mode == 0 ? 4 : 2;
  double acc = 0.0;  // warp w < nterm: term w of row r0 + lane
  for (int i0 = 0; i0 < ni; i0 += 32) {
    for (int rr = w; rr < RS_ROWS; rr += 8) {
      const int r = r0 + rr;
      if (r < nr && i0 + lane < ni) {
        const int j = G.js + r % nj, k = G.ks + (r / nj) % nk, b = r / (nj * nk);
        const DevBlock& B = blks[b];
        double* const* U = B.st[0];
        const int id = G.idx(k, j, G.is + i0 + lane);
        const double rho = U[0][id];
        const double d0 = B.fx[0][0][id], d1 = B.fx[0][1][id], d2 = B.fx[0][2][id];
        if (mode == 0) {
          term[0][rr][lane] = rho;
          term[1][rr][lane] = rho * d0;
          term[2][rr][lane] = rho * d1;
          term[3][rr][lane] = rho * d2;
        } else {
          const double p0 = d0 - m0, p1 = d1 - m1, p2 = d2 - m2;
          const double q = p0 * p0 + p1 * p1 + p2 * p2;
          term[0][rr][lane] = 0.5 * rho * q;
          term[1][rr][lane] = U[1][id] * p0 + U[2][id] * p1 + U[3][id] * p2;
        }
      }
    }
    __syncthreads();
    if (w < nterm) {
      const int n = min(32, ni - i0);
      for (int c = 0; c < n; ++c) acc = acc + term[w][lane][c];
    }
    __syncthreads();
  }
  if (r0 + lane < nr && w < 4) rows[4 * (r0 + lane) + w] = (w < nterm) ? acc : 0.0;
}

// per (block, k) plane: its rows summed in j order; then per block: its
// planes summed in k order
__global__ void k_drive_planes(KGeom G, const double* __restrict__ rows, double* planes) {
  const int nj = G.je - G.js, nk = G.ke - G.ks;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 4 * G.nb * nk) return;
  const int q = t & 3, p = t >> 2;
  const double* r = rows + 4 * (long long)p * nj + q;
  double s = 0.0;
  for (int j = 0; j < nj; ++j) s = s + r[4 * j];
  planes[t] = s;
}

__global__ void k_drive_blocks(KGeom G, const double* __restrict__ planes, double* sums) {
  const int nk = G.ke - G.ks;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 4 * G.nb) return;
  const int q = t & 3, b = t >> 2;
  const double* p = planes + 4 * (long long)b * nk + q;
  double s = 0.0;
  for (int k = 0; k < nk; ++k) s = s + p[4 * k];
  sums[t] = s;
}

// m += (s rho) dv', E += KE(m_new) - KE(m) on every active cell
__global__ void k_drive_apply(const DevBlock* __restrict__ blks, KGeom G, double m0, double m1, double m2,
                              double scale) {
  const int ni = G.ie - G.is, nj = G.je - G.js, nk = G.ke - G.ks;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)G.nb * nk * nj * ni) return;
  const int i = G.is + (int)(t % ni);
  const int j = G.js + (int)((t / ni) % nj);
  const int k = G.ks + (int)((t / ((long long)ni * nj)) % nk);
  const int b = (int)(t / ((long long)ni * nj * nk));
  const DevBlock& B = blks[b];
  double* const* U = B.st[0];
  const int id = G.idx(k, j, i);
  const double rho = U[0][id];
  const double p0 = B.fx[0][0][id] - m0, p1 = B.fx[0][1][id] - m1, p2 = B.fx[0][2][id] - m2;
  const double a0 = U[1][id], a1 = U[2][id], a2 = U[3][id];
  const double sr = scale * rho;
  const double n0 = a0 + sr * p0, n1 = a1 + sr * p1, n2 = a2 + sr * p2;
  const double irho = 1.0 / rho;
  const double ke0 = 0.5 * (a0 * a0 + a1 * a1 + a2 * a2) * irho;
  const double ke1 = 0.5 * (n0 * n0 + n1 * n1 + n2 * n2) * irho;
  U[1][id] = n0;
  U[2][id] = n1;
  U[3][id] = n2;
  U[4][id] = U[4][id] + (ke1 - ke0);
}

}  // namespace

void launch_drive_dv(const DevBlock* blks, const KGeom& G, const DriveTabs& T, cudaStream_t s) {
  const int nkr = (G.ke - G.ks + DV_KC - 1) / DV_KC;
  const long long n = (long long)G.nb * nkr * (G.je - G.js) * (G.ie - G.is);
  k_drive_dv<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(blks, G, T);
}

// rows: nb x nk x nj x 4 row sums followed by nb x nk x 4 plane sums
void launch_drive_sums(const DevBlock* blks, const KGeom& G, int mode, const double mean[3], double* rows,
                       double* sums, cudaStream_t s) {
  const int nr = G.nb * (G.ke - G.ks) * (G.je - G.js);
  const int npl = G.nb * (G.ke - G.ks);
  double* planes = rows + 4 * (size_t)nr;
  k_drive_rows<<<(nr + RS_ROWS - 1) / RS_ROWS, 256, 0, s>>>(blks, G, mode, mean[0], mean[1], mean[2], rows);
  k_drive_planes<<<(4 * npl + 127) / 128, 128, 0, s>>>(G, rows, planes);
  k_drive_blocks<<<(4 * G.nb + 127) / 128, 128, 0, s>>>(G, planes, sums);
}

void launch_drive_apply(const DevBlock* blks, const KGeom& G, const double mean[3], double scale,
                        cudaStream_t s) {
  const long long n = (long long)G.nb * (G.ke - G.ks) * (G.je - G.js) * (G.ie - G.is);
  k_drive_apply<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(blks, G, mean[0], mean[1], mean[2], scale);
}

}  // namespace pmhd_gpu
