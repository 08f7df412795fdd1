// kernels_halo.cu -- pack / unpack of the ghost + face-B halo slabs that cross
// a rank boundary (pack_boundary / unpack_boundary).
//
// Buffer layout (identical to the oracle's pack/unpack): variable-major
// (u0..u4, b1f, b2f, b3f), each slab in k-j-i order with i fastest.  One
// launch moves one slab message between a block's arrays and a contiguous
// device buffer that the caller hands to NCCL send/recv (or any transport).
#include "kernels.cuh"

namespace pmhd_gpu {

namespace {

__global__ void k_halo_copy(double* const* arrays, KGeom G, HaloSlab sl, double* buf, int to_buf) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= sl.off[8]) return;
  int v = 0;
#pragma unroll
  for (int q = 1; q < 8; ++q) v += (t >= sl.off[q]) ? 1 : 0;
  const long long l = t - sl.off[v];
  const int ni = sl.ext[v][0], nj = sl.ext[v][1];
  const int i = sl.org[v][0] + (int)(l % ni);
  const int j = sl.org[v][1] + (int)((l / ni) % nj);
  const int k = sl.org[v][2] + (int)(l / ((long long)ni * nj));
  const int id = G.idx(k, j, i);
  if (to_buf) buf[t] = arrays[v][id];
  else arrays[v][id] = buf[t];
}

// Dense host-order array (e1 x e2 x e3, i fastest) <-> pitched block array:
// upload / download stage through a contiguous device buffer so the PCIe
// transfer is one large DMA instead of a 3D copy of 2 KB rows.
__global__ void k_repack(double* dense, double* pitched, KGeom G, int e1, int e2, int e3,
                         int to_dense) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)e1 * e2 * e3) return;
  const int i = (int)(t % e1);
  const int j = (int)((t / e1) % e2);
  const int k = (int)(t / ((long long)e1 * e2));
  const int id = G.idx(k, j, i);
  if (to_dense) dense[t] = pitched[id];
  else pitched[id] = dense[t];
}

// face_to_center_b of component c into a dense n1 x n2 x n3
// array (same IEEE operations as the oracle: 0.5 * (lo + hi)).
__global__ void k_bcc_dense(double* dense, const double* bf, KGeom G, int c) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)G.n1 * G.n2 * G.n3) return;
  const int i = (int)(t % G.n1);
  const int j = (int)((t / G.n1) % G.n2);
  const int k = (int)(t / ((long long)G.n1 * G.n2));
  const int id = G.idx(k, j, i);
  const int off = (c == 0) ? 1 : ((c == 1) ? G.sx : G.sy);
  dense[t] = 0.5 * (bf[id] + bf[id + off]);
}

}  // namespace

void launch_repack(double* dense, double* pitched, const KGeom& G, int e1, int e2, int e3,
                   int to_dense, cudaStream_t s) {
  const long long n = (long long)e1 * e2 * e3;
  if (n <= 0) return;
  k_repack<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dense, pitched, G, e1, e2, e3, to_dense);
}

void launch_bcc_dense(double* dense, const double* bf, const KGeom& G, int c, cudaStream_t s) {
  const long long n = (long long)G.n1 * G.n2 * G.n3;
  k_bcc_dense<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dense, bf, G, c);
}

void launch_halo_copy(double* const* dev_arrays, const KGeom& G, const HaloSlab& sl, double* buf,
                      int to_buf, cudaStream_t s) {
  const long long n = sl.off[8];
  if (n <= 0) return;
  k_halo_copy<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dev_arrays, G, sl, buf, to_buf);
}

}  // namespace pmhd_gpu
