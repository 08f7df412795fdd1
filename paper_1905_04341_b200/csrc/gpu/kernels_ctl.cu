// kernels_ctl.cu -- one-thread control kernels of a graph-replayed run: the
// stage coefficients written on the device (the fused kernels' MODE 2 reads
// them, so a cycle is captured once and replayed as a CUDA graph), and the cycle loop of
// pmhd_gpu_run (dt from the stage-2 reduction, the tlim cap of SPEC.md:256,
// error / floor bookkeeping) kept on the device between graph replays.  The
// arithmetic is the host's (same IEEE operations), so a replayed run is bit
// for bit the host-driven one.
#include <climits>

#include "kernels.cuh"

namespace pmhd_gpu {

namespace {

__device__ void stage_coeffs(KStage& k, int s, double h, const double* dx) {
  const double beta = (s == 1) ? 0.5 : 1.0;
  const double bdt = beta * h;
  k.c1 = bdt / dx[0];
  k.c2 = bdt / dx[1];
  k.c3 = bdt / dx[2];
  for (int d = 0; d < 3; ++d) k.c1024[d] = 1024.0 * h / dx[d];
  k.in_sel = (s == 1) ? 0 : 1;
  k.out_sel = (s == 1) ? 1 : 2;
  k.stage = s;
  k.plm = (s == 2);
  k.skip = 0;
}

__global__ void k_cycle_begin(DevCtl* ctl, KStage* dks, DevRed* red) {
  if (ctl->stop) {
    dks[1].skip = 1;
    dks[2].skip = 1;
    return;
  }
  double h = ctl->dt;
  int last = 0;
  if (ctl->tlim > 0.0 && ctl->t + h >= ctl->tlim) {  // land exactly on tlim
    h = ctl->tlim - ctl->t;
    last = 1;
  }
  ctl->h = h;
  ctl->last = last;
  stage_coeffs(dks[1], 1, h, ctl->dx);
  stage_coeffs(dks[2], 2, h, ctl->dx);
  for (int q = 0; q < 3; ++q) {
    red[q].dt_bits = 0x7FF0000000000000ULL;  // +inf
    red[q].bad_key = ULLONG_MAX;
    red[q].floor_count = 0;
    red[q].divb_bits = 0;
    red[q].fallback_count = 0;
    for (int p = 0; p < 5; ++p) red[q].phase[p] = 0;
  }
}

__global__ void k_cycle_end(DevCtl* ctl, const KStage* dks, const DevRed* red) {
  if (dks[1].skip) return;  // this cycle did not run
  const unsigned long long fl = red[1].floor_count + red[2].floor_count;
  const unsigned long long fb = red[1].fallback_count + red[2].fallback_count;
  if (red[1].bad_key != ULLONG_MAX || red[2].bad_key != ULLONG_MAX) {
    ctl->err_stage = (red[1].bad_key != ULLONG_MAX) ? 1 : 2;
    ctl->err_key = (ctl->err_stage == 1) ? red[1].bad_key : red[2].bad_key;
    ctl->err_floors = fl;
    ctl->stop = 1;
    return;
  }
  ctl->floors += fl;
  ctl->fallbacks += fb;
  ctl->t = ctl->last ? ctl->tlim : ctl->t + ctl->h;
  ctl->dt = ctl->cfl * __longlong_as_double((long long)red[0].dt_bits);
  ctl->cycles += 1;
  if ((ctl->ncycles >= 0 && ctl->cycles >= ctl->ncycles) || (ctl->tlim > 0.0 && ctl->t >= ctl->tlim))
    ctl->stop = 1;
}

}  // namespace


void launch_cycle_begin(DevCtl* ctl, KStage* dks, DevRed* red, cudaStream_t s) {
  k_cycle_begin<<<1, 1, 0, s>>>(ctl, dks, red);
}

void launch_cycle_end(DevCtl* ctl, const KStage* dks, const DevRed* red, cudaStream_t s) {
  k_cycle_end<<<1, 1, 0, s>>>(ctl, dks, red);
}

}  // namespace pmhd_gpu
