// kernels_drive.cu -- turbulence driving (the "driven" phase
// of BASELINE config 5): an impulsive solenoidal velocity kick every
// turb_every cycles (definition in include/pmhd_host.h, oracle restatement
// in oracle/pmhd_oracle.hpp drive_*).  The global sums it needs are formed
// in a fixed order -- each (k, j) row summed over i by one thread, the rows of
// a block summed in (k, j) order by one thread, blocks combined on the host
// in gid order -- so one process, several ranks and the CPU oracle agree bit
// for bit.  Runs once per driving event, not on the timed VL2 path.
#include "kernels.cuh"

namespace pmhd_gpu {

namespace {

__device__ __forceinline__ int gidx(const KGeom& G, const DevBlock& B, int a, int l) {
  // global cell index along axis a of local index l
  const int s = (a == 0) ? G.is : (a == 1 ? G.js : G.ks);
  return B.c[a] * G.mb[a] + (l - s);
}

// dv = sum_m c_m cos(k.x) + s_m sin(k.x) on every active cell -> B.fx[0][0..2]
__global__ void k_drive_dv(const DevBlock* __restrict__ blks, KGeom G, DriveTabs T) {
  const int ni = G.ie - G.is, nj = G.je - G.js, nk = G.ke - G.ks;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)G.nb * nk * nj * ni) return;
  const int i = G.is + (int)(t % ni);
  const int j = G.js + (int)((t / ni) % nj);
  const int k = G.ks + (int)((t / ((long long)ni * nj)) % nk);
  const int b = (int)(t / ((long long)ni * nj * nk));
  const DevBlock& B = blks[b];
  const int gi = gidx(G, B, 0, i), gj = gidx(G, B, 1, j), gk = (G.dim == 3) ? gidx(G, B, 2, k) : 0;
  double dv0 = 0.0, dv1 = 0.0, dv2 = 0.0;
  for (int m = 0; m < T.n; ++m) {
    const int qx = (T.k[m][0] + 2) * G.nx[0] + gi;
    const int qy = (T.k[m][1] + 2) * G.nx[1] + gj;
    const int qz = (T.k[m][2] + 2) * G.nx[2] + gk;
    const double axr = T.ct[0][qx], axi = T.st[0][qx];
    const double ayr = T.ct[1][qy], ayi = T.st[1][qy];
    const double azr = T.ct[2][qz], azi = T.st[2][qz];
    const double zr = axr * ayr - axi * ayi, zi = axr * ayi + axi * ayr;
    const double cr = zr * azr - zi * azi, ci = zr * azi + zi * azr;
    dv0 = dv0 + (T.c[m][0] * cr + T.s[m][0] * ci);
    dv1 = dv1 + (T.c[m][1] * cr + T.s[m][1] * ci);
    dv2 = dv2 + (T.c[m][2] * cr + T.s[m][2] * ci);
  }
  const int id = G.idx(k, j, i);
  B.fx[0][0][id] = dv0;
  B.fx[0][1][id] = dv1;
  B.fx[0][2][id] = dv2;
}

// per (block, k, j) row, summed over i in order.  mode 0: (rho, rho dv);
// mode 1: (1/2 rho |dv'|^2, m.dv') with dv' = dv - mean
__global__ void k_drive_rows(const DevBlock* __restrict__ blks, KGeom G, int mode, double m0, double m1,
                             double m2, double* rows) {
  const int nj = G.je - G.js, nk = G.ke - G.ks;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= G.nb * nk * nj) return;
  const int j = G.js + t % nj, k = G.ks + (t / nj) % nk, b = t / (nj * nk);
  const DevBlock& B = blks[b];
  double* const* U = B.st[0];
  double r0 = 0.0, r1 = 0.0, r2 = 0.0, r3 = 0.0;
  for (int i = G.is; i < G.ie; ++i) {
    const int id = G.idx(k, j, i);
    const double rho = U[0][id];
    const double d0 = B.fx[0][0][id], d1 = B.fx[0][1][id], d2 = B.fx[0][2][id];
    if (mode == 0) {
      r0 = r0 + rho;
      r1 = r1 + rho * d0;
      r2 = r2 + rho * d1;
      r3 = r3 + rho * d2;
    } else {
      const double p0 = d0 - m0, p1 = d1 - m1, p2 = d2 - m2;
      const double q = p0 * p0 + p1 * p1 + p2 * p2;
      r0 = r0 + 0.5 * rho * q;
      r1 = r1 + (U[1][id] * p0 + U[2][id] * p1 + U[3][id] * p2);
    }
  }
  rows[4 * t + 0] = r0;
  rows[4 * t + 1] = r1;
  rows[4 * t + 2] = r2;
  rows[4 * t + 3] = r3;
}

// per block: its rows summed in (k, j) order
__global__ void k_drive_blocks(KGeom G, const double* rows, double* sums) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= G.nb) return;
  const int nr = (G.ke - G.ks) * (G.je - G.js);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int r = 0; r < nr; ++r) {
    const double* q = rows + 4 * ((long long)b * nr + r);
    s0 = s0 + q[0];
    s1 = s1 + q[1];
    s2 = s2 + q[2];
    s3 = s3 + q[3];
  }
  sums[4 * b + 0] = s0;
  sums[4 * b + 1] = s1;
  sums[4 * b + 2] = s2;
  sums[4 * b + 3] = s3;
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
  const long long n = (long long)G.nb * (G.ke - G.ks) * (G.je - G.js) * (G.ie - G.is);
  k_drive_dv<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(blks, G, T);
}

void launch_drive_sums(const DevBlock* blks, const KGeom& G, int mode, const double mean[3], double* rows,
                       double* sums, cudaStream_t s) {
  const int nr = G.nb * (G.ke - G.ks) * (G.je - G.js);
  k_drive_rows<<<(nr + 127) / 128, 128, 0, s>>>(blks, G, mode, mean[0], mean[1], mean[2], rows);
  k_drive_blocks<<<(G.nb + 63) / 64, 64, 0, s>>>(G, rows, sums);
}

void launch_drive_apply(const DevBlock* blks, const KGeom& G, const double mean[3], double scale,
                        cudaStream_t s) {
  const long long n = (long long)G.nb * (G.ke - G.ks) * (G.je - G.js) * (G.ie - G.is);
  k_drive_apply<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(blks, G, mean[0], mean[1], mean[2], scale);
}

}  // namespace pmhd_gpu
