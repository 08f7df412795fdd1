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

}  // namespace

void launch_halo_copy(double* const* dev_arrays, const KGeom& G, const HaloSlab& sl, double* buf,
                      int to_buf, cudaStream_t s) {
  const long long n = sl.off[8];
  if (n <= 0) return;
  k_halo_copy<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dev_arrays, G, sl, buf, to_buf);
}

}  // namespace pmhd_gpu
