// kernels.cuh -- device data layout shared by the ABI and the kernels.
//
// HBM layout: every per-block field is a dense
// k-j-i array (i fastest, the reference's Array3 order, array.hpp:30-35) with
// a padded row pitch sx (multiple of 32 doubles = 256 B) and a plane pitch
// sy = sx * (n2 + 1), so cell-, face- and edge-centred arrays share one index
// function idx(k,j,i) = k*sy + j*sx + i.  Variables are separate arrays
// (variable-major, array.hpp:61-66).
#ifndef PMHD_KERNELS_CUH_
#define PMHD_KERNELS_CUH_

#include <cuda.h>  // CUtensorMap (type only; maps are encoded through the runtime's driver entry point)
#include <cuda_runtime.h>

#include "physics.cuh"

namespace pmhd_gpu {

constexpr int kNState = 8;  // u0..u4 (rho, m1, m2, m3, E), b1f, b2f, b3f

struct KGeom {
  int n1, n2, n3;     // cell extents incl. ghosts
  int sx, sy;         // row / plane pitch (doubles; a block array is < 2^31 doubles)
  int is, ie, js, je, ks, ke;
  int dim, nb, ng;
  int nx[3], mb[3];
  double dx[3];
  __host__ __device__ int idx(int k, int j, int i) const { return k * sy + j * sx + i; }
};

// Bounds-checked debug build (-DPMHD_BOUNDS_CHECK, lib/test/libpmhd_gpu_check.so;
// compute-sanitizer is not available on the GPU pool): every element index the
// fused kernels and the exchange form into a block array must lie inside the
// array's (n3+1) planes, else the kernel traps.
#ifdef PMHD_BOUNDS_CHECK
#define PMHD_CHECK_ID(G, id)                                                  \
  do {                                                                        \
    if ((unsigned)(id) >= (unsigned)(((G).n3 + 1) * (G).sy)) __trap();       \
  } while (0)
#else
#define PMHD_CHECK_ID(G, id) \
  do {                       \
  } while (0)
#endif

struct DevBlock {
  // st[0] = u^n (current), st[1] = u^{n+1/2}, st[2] = u^{n+1} (next).  The
  // ABI keeps two device copies of the block table with st[0] and st[2]
  // swapped and flips between them after each cycle, so no stage updates a
  // buffer that another tile still reads (tiles recompute shared faces).
  double* st[3][kNState];
  double* w[8];            // stage-input primitives incl. Bcc (split kernels)
  double* fx[3][8];        // face data: 5 lab-order fluxes, ey, ez, weight
  double* e[3];            // corner EMFs e1, e2, e3 (split kernels)
  double* ec[3];           // cell-centred E = -v x B of the stage input (fused
                           // kernels; aliases e[], which they do not use)
  int c[3];                // block coordinates
  int nbr[3][2];           // local index of the lower / upper neighbour
  // peer-memory halo (pmhd_gpu_peer_attach): this block's base in its slab
  // and, for a neighbour owned by another rank on the node, that block's base
  // as mapped into this process (CUDA IPC over NVLink); an array of the
  // neighbour is at rbase + (own array - base) (same layout on every rank)
  const char* base;
  const char* rbase[3][2];
};

// Device-side reduction slots: red[0] = init / dt, red[1..2] = stage 1..2.
struct DevRed {
  unsigned long long dt_bits;     // min over cells of dx/(|v|+cf), as bits
  unsigned long long bad_key;     // smallest failing global cell key
  unsigned long long floor_count;
  unsigned long long divb_bits;   // max |div B| as bits
  unsigned long long fallback_count;  // Roe -> HLLE fallbacks
  // profiling only (KPhys::prof): SM cycles summed over CTAs per kernel phase
  // -- flux: [0] load + cons_to_prim, [1] reconstruct, [2] Riemann;
  // update: [3] Ec + corner EMFs, [4] CT + conserved update + c2p + dt
  unsigned long long phase[5];
};

// Stage coefficients c_d = beta*dt/dx_d, computed on the host with the same
// IEEE operations as the oracle.
// Stage coefficients: by value, or (graph-replayed runs, kernel MODE 2) from
// the device copy k_cycle_begin writes, so a captured cycle can be replayed.
// skip != 0: the replayed cycle is past the end of the run; kernels return.
struct KStage {
  double c1, c2, c3;
  double c1024[3];  // 1024 * dt / dx_d (contact-upwind weight scale)
  int in_sel, out_sel, stage, plm;  // base is always st[0]
  int skip;
};

// Device-resident run control (graph-replayed pmhd_gpu_run): the cycle loop
// of the ABI's run (dt cap to land on tlim) without a host
// round trip per cycle.
struct DevCtl {
  double t, dt, tlim, h, cfl;
  double dx[3];
  int last, stop, cycles, ncycles;
  unsigned long long floors, fallbacks;      // completed cycles
  unsigned long long err_key, err_floors;    // failing cycle (stop with an error)
  int err_stage, pad;
};
void launch_cycle_begin(DevCtl* ctl, KStage* dks, DevRed* red, cudaStream_t s);
void launch_cycle_end(DevCtl* ctl, const KStage* dks, const DevRed* red, cudaStream_t s);

// One halo slab message: per array v, its origin and extents (i, j, k) and its
// offset in the contiguous buffer (off[8] = total doubles).
struct HaloSlab {
  int org[8][3];
  int ext[8][3];
  long long off[9];
};
void launch_halo_copy(double* const* dev_arrays, const KGeom& G, const HaloSlab& sl, double* buf,
                      int to_buf, cudaStream_t s);
// Turbulence driving (kernels_drive.cu): device copies of the modes and the
// per-axis phase tables (pmhd_host.h pmhd_drive_modes / drive_tables).
struct DriveTabs {
  int n;
  int k[64][3];
  double c[64][3], s[64][3];
  const double* ct[3];  // cos tables, (k+2)*nx[a] + g
  const double* st[3];  // sin tables
};
void launch_drive_dv(const DevBlock* blks, const KGeom& G, const DriveTabs& T, cudaStream_t s);
void launch_drive_sums(const DevBlock* blks, const KGeom& G, int mode, const double mean[3], double* rows,
                       double* sums, cudaStream_t s);
void launch_drive_apply(const DevBlock* blks, const KGeom& G, const double mean[3], double scale,
                        cudaStream_t s);
void launch_repack(double* dense, double* pitched, const KGeom& G, int e1, int e2, int e3,
                   int to_dense, cudaStream_t s);
void launch_bcc_dense(double* dense, const double* bf, const KGeom& G, int c, cudaStream_t s);

// Launchers (kernels.cu).
void launch_c2p_all(const DevBlock* blks, const KGeom& G, const KPhys& ph, int sel, DevRed* red,
                    int stage, cudaStream_t s);
void launch_flux(const DevBlock* blks, const KGeom& G, const KPhys& ph, int dir, int sel, int plm,
                 double c1024, cudaStream_t s);
// Kernel choices of the flux launcher, read from the PMHD_* environment at
// mesh creation (pmhd_gpu_mesh_create)
struct FluxOpts {
  int reuse = 0;     // owned-face ranges + rim images (PMHD_FACE_REUSE)
  int march = 1;     // x2 / x3 column march: 0 off, 1 where it fills the GPU, 2 always (PMHD_FLUX_MARCH)
  int march_x1 = 1;  // x1 row march too (PMHD_FLUX_MARCH_X1)
  // bit s-1: the march kernels in stage s (PMHD_FLUX_MARCH_STAGES): stage 2
  // only -- with donor-cell states (stage 1) the tile kernels are as fast or
  // faster, with PLM (stage 2) the marches win
  int march_stages = 2;
  int pad = 0;       // experiment: unused dynamic shared memory per tile CTA, bytes (PMHD_FLUX_SMEM_PAD)
};
// region: 0 all tiles, 1 tiles clear of the ghost exchange, 2 the others
// kd: nullptr (coefficients by value) or the device copy of a graph-replayed cycle
void launch_flux_fused(const DevBlock* blks, const KGeom& G, const KPhys& ph, int dir, int sel,
                       int plm, double c1024, const KStage* kd, int stage, DevRed* red, int slab,
                       int nslab, int S, cudaStream_t s, int region = 0, const FluxOpts& opt = FluxOpts());
// x1 and x2 faces in one launch (owned-face ranges; kernels_flux.cu k_flux_xy)
void launch_flux_xy(const DevBlock* blks, const KGeom& G, const KPhys& ph, int sel, int plm, double c1024x,
                    double c1024y, const KStage* kd, int stage, DevRed* red, cudaStream_t s);
void launch_emf(const DevBlock* blks, const KGeom& G, const KPhys& ph, cudaStream_t s);
// ec_maps (optional, 3D meshes): per block, TMA tensor maps of its 3 cell-E
// arrays (box = the update tile's E box) -- the kernel then streams its E
// ring with TMA, one plane ahead.  Box extents: update_ec_box().
void launch_update_fused(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks,
                         const KStage* kd, DevRed* red, int want_dt, int kr0, int kr1, cudaStream_t s,
                         const CUtensorMap* ec_maps = nullptr, int push = 0);
void update_ec_box(int box[2]);
// TMA-staged update kernel (kernels_update_tma.cu, 3D meshes): maps[b * per
// block + id] are the tensor maps of block b for the table the launch uses;
// bit id of xoffm = 1 when that map starts one element before its array (16 B
// alignment of the map base).
// warp-specialised update kernel (kernels_update_ws.cu, 3D)
// Two barrier-free kernels (corner EMFs, then CT + conserved update + c2p + dt;
// in 2D only E3 is formed): the corner EMFs go through the block's w[0..2]
// arrays.  The default where update_emf_fills (every mesh unless built with
// PMHD_EMF_SMALL=0; PMHD_UPDATE=emf: always, =ldg: never).
bool update_emf_fills(const KGeom& G, int kr0, int kr1);
void launch_update_emf(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks,
                       const KStage* kd, DevRed* red, int want_dt, int kr0, int kr1, cudaStream_t s, int push,
                       int all_local);
void launch_update_ws(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks, const KStage* kd,
                      DevRed* red, int want_dt, int kr0, int kr1, cudaStream_t s, int push);
int update_tma_maps_per_block();
void update_tma_box(int id, int box[3]);  // width, height, first cell rel. to the tile origin
const double* update_tma_array(const DevBlock& B, int id);
void launch_update_tma(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks,
                       const KStage* kd, DevRed* red, int want_dt, int kr0, int kr1, cudaStream_t s,
                       const CUtensorMap* maps, unsigned long long xoffm, int push);
bool update_uses_tma();  // built with PMHD_UPDATE_TMA
void launch_update(const DevBlock* blks, const KGeom& G, const KStage& ks, cudaStream_t s);
void launch_c2p_end(const DevBlock* blks, const KGeom& G, const KPhys& ph, const KStage& ks,
                    DevRed* red, int want_dt, cudaStream_t s);
// kd (optional): skip flag of a graph-replayed cycle
void launch_exchange(const DevBlock* blks, const KGeom& G, int sel, cudaStream_t s,
                     const KStage* kd = nullptr);
void launch_exchange_dir(const DevBlock* blks, const KGeom& G, int sel, int dir, cudaStream_t s,
                         const KStage* kd = nullptr);
void launch_dt_from_state(const DevBlock* blks, const KGeom& G, const KPhys& ph, DevRed* red,
                          cudaStream_t s);
void launch_divb(const DevBlock* blks, const KGeom& G, DevRed* red, cudaStream_t s);
void launch_row_sums(const DevBlock* blks, const KGeom& G, double* rows, cudaStream_t s);

}  // namespace pmhd_gpu

#endif
