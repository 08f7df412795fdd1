/*
 * pmhd_gpu.h -- C ABI of the B200 (sm_100a) VL2+PLM+HLLD/HLLE+CT MHD update.
 *
 * This is the drop-in boundary for the reference's hot path.  In the reference
 * the path is a set of C++ ops executed through the exec layer:
 *   par_for / par_reduce          /root/reference/proj/include/pmhd/exec/dispatch.hpp:109-143
 *   vl2_step
 *   exchange_ghosts
 *   compute_dt
 *   cons_to_prim / face_to_center_b
 *   max_divergence_b
 * Lambdas cannot cross a C ABI, so the seam sits one level up, at the solver
 * ops that cmd_run / cmd_bench / cmd_scale call.  Each entry
 * point below names the reference op it replaces.
 *
 * Conventions
 *  - All arithmetic is fp64 (Real=double, defs.hpp:16).  The parity library
 *    (libpmhd_gpu_parity.so) uses IEEE operations in the oracle's order and
 *    is bit-identical to the CPU oracle.  The product library
 *    (libpmhd_gpu.so) contracts multiply-adds into FMAs and forms division
 *    and square root within 1 ulp of the IEEE result (INTEGRATION.md
 *    section 4); its fields stay within 1e-11 per cell of the oracle.
 *  - Host arrays are exactly the reference layout (array.hpp:19-80): k-j-i
 *    order with i fastest; the conserved array is variable-major with
 *    NCONS=8 variables (rho,m1,m2,m3,E,Bcc1,Bcc2,Bcc3; defs.hpp:22).  Block
 *    arrays include ng ghost layers on every side of every dimension that has
 *    more than one cell (nx3==1 => 2D, no x3 ghosts).  Face arrays are one
 *    larger in their own dimension.
 *  - Indices are half-open [is,ie) (loop.hpp:17).
 *  - Every call returns 0 (PMHD_OK) or one of the PMHD_ERR_* codes, which
 *    mirror the exception types of defs.hpp:36-76.  No C++ exception crosses
 *    the ABI.  pmhd_gpu_last_error() returns a message for the last failure.
 *  - A context is driven by one host thread (profiler.hpp:8-10); calls are not
 *    re-entrant.  Each call returns once its results are visible to the next
 *    call (dispatch.hpp:106-108 synchronization-point semantics).
 *  - There is no CPU fallback: creating a context without a usable sm_100
 *    device fails with PMHD_ERR_CUDA.
 */
#ifndef PMHD_GPU_H_
#define PMHD_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMHD_ABI_VERSION 1

/* Error codes (defs.hpp:36-76). */
enum {
  PMHD_OK = 0,
  PMHD_ERR_CONFIG = 1,      /* ConfigError          defs.hpp:36-39 */
  PMHD_ERR_BUFFER = 2,      /* BufferError          defs.hpp:41-44 */
  PMHD_ERR_INPUT = 3,       /* InputError           defs.hpp:46-49 */
  PMHD_ERR_UNPHYSICAL = 4,  /* UnphysicalStateError defs.hpp:51-62 */
  PMHD_ERR_CUDA = 5,        /* device / driver failure (no reference analogue) */
  PMHD_ERR_UNSUPPORTED = 6  /* UnsupportedKernelError defs.hpp:72-76 */
};

/* Riemann solvers (north_star: HLLD and HLLE). */
enum { PMHD_RIEMANN_HLLD = 0, PMHD_RIEMANN_HLLE = 1,
       PMHD_RIEMANN_ROE = 2 /* SPEC.md:177-185, HLLE fallback counted */ };
/* PLM slope limiters (MC; van Leer selectable). */
enum { PMHD_LIMITER_MC = 0, PMHD_LIMITER_VANLEER = 1 };
/* cons->prim failure policy (SPEC.md:136 error; Athena++-style floors). */
enum { PMHD_EOS_ERROR = 0, PMHD_EOS_FLOOR = 1 };
/* Corner-EMF average (contact-upwind; 4-point mean behind a flag). */
enum { PMHD_EMF_UPWIND = 0, PMHD_EMF_ARITH = 1 };
/* Diagnostics for pmhd_gpu_diag. */
enum {
  PMHD_DIAG_DIVB_MAX = 0, /* max_divergence_b: out[0]            */
  PMHD_DIAG_SUMS = 1      /* sum over active cells of the 5 hydro conserved vars
                             (fixed-order per block, blocks in gid order): out[0..4] */
};

/* Mesh descriptor: MeshConfig plus solver options. */
typedef struct pmhd_mesh_desc {
  int nx[3];          /* global active cells per dimension (nx[2]==1 => 2D)   */
  int mb[3];          /* MeshBlock active cells per dimension                 */
  int ng;             /* ghost width, >= 2                                     */
  double xmin[3];     /* physical domain                                       */
  double xmax[3];
  double gamma;       /* adiabatic index, > 1                                  */
  double cfl;         /* CFL number in (0,1)                                   */
  int riemann;        /* PMHD_RIEMANN_*                                        */
  int limiter;        /* PMHD_LIMITER_*                                        */
  int eos_mode;       /* PMHD_EOS_*                                            */
  int emf_mode;       /* PMHD_EMF_*                                            */
  double dfloor;      /* density floor   (eos_mode == FLOOR)                   */
  double pfloor;      /* pressure floor  (eos_mode == FLOOR)                   */
} pmhd_mesh_desc;

/* Per-call solver status (UnphysicalStateError payload, defs.hpp:51-62). */
typedef struct pmhd_status {
  int code;               /* PMHD_OK or PMHD_ERR_UNPHYSICAL                     */
  int stage;              /* 1 or 2 (SPEC.md:213 stage tag); 0 = init / dt      */
  int k, j, i;            /* lexicographically smallest failing GLOBAL active cell */
  long long floor_count;  /* floor activations in this call (eos_mode FLOOR)   */
  long long fallback_count; /* faces where Roe fell back to HLLE */
} pmhd_status;

/* Region times (Fig. 3 analogue), milliseconds accumulated since
 * the last reset, measured with CUDA events on the solver stream. */
typedef struct pmhd_region_times {
  double c2p_ms, riemann_ms, ct_emf_ms, integrate_ms, boundary_ms, dt_ms;
  long long calls;           /* profiled stages                               */
  long long kernel_launches; /* kernels this library launched (always counted) */
  /* reconstruction ("reconstruct").  The fused kernels' event
   * times are split into c2p / reconstruct / riemann and ct_emf / integrate
   * by the SM-cycle shares of their phases (clock64 at the kernel barriers). */
  double reconstruct_ms;
} pmhd_region_times;

typedef struct pmhd_ctx pmhd_ctx;
typedef struct pmhd_mesh pmhd_mesh;

/* ABI version; a host binding checks it before any other call. */
int pmhd_gpu_abi_version(void);

/* Context on one CUDA device (one process per GPU).  Fails with
 * PMHD_ERR_CUDA if the device is absent or not sm_100. */
int pmhd_gpu_ctx_create(int device, pmhd_ctx** out);
int pmhd_gpu_ctx_destroy(pmhd_ctx* ctx);
/* Message describing the last failure on this context (never NULL). */
const char* pmhd_gpu_last_error(const pmhd_ctx* ctx);

/* build_mesh restricted to the blocks this context owns.
 * gids: the global block ids held by this context (lexicographic block order,
 * i fastest); n_local <= 0 means "all blocks".  Validation errors mirror
 * MeshConfig invariants -> PMHD_ERR_CONFIG. */
int pmhd_gpu_mesh_create(pmhd_ctx* ctx, const pmhd_mesh_desc* desc, const int* gids,
                         int n_local, pmhd_mesh** out);
int pmhd_gpu_mesh_destroy(pmhd_mesh* mesh);

/* Block array extents (with ghosts): n[0]=n1, n[1]=n2, n[2]=n3. */
int pmhd_gpu_block_dims(const pmhd_mesh* mesh, int n[3]);

/* Copy a block's state in.  u: NCONS x n3 x n2 x n1 (Bcc entries are ignored:
 * they are owned by the face fields, defs.hpp:18-21); b1f: n3 x n2 x (n1+1);
 * b2f: n3 x (n2+1) x n1; b3f: (n3+1) x n2 x n1.  All pointers are host memory,
 * borrowed for the call. */
int pmhd_gpu_upload_block(pmhd_mesh* mesh, int gid, const double* u, const double* b1f,
                          const double* b2f, const double* b3f);
/* Copy a block's state out.  u receives the 5 hydro variables and Bcc from
 * face_to_center_b; w (may be NULL) receives cons_to_prim of
 * every cell incl. ghosts (rho,v1,v2,v3,p,Bcc1..3); any pointer may be NULL. */
int pmhd_gpu_download_block(pmhd_mesh* mesh, int gid, double* u, double* w, double* b1f,
                            double* b2f, double* b3f);

/* exchange_ghosts: periodic x1 -> x2 -> x3 sweeps over the
 * blocks of this mesh (all blocks must be local). */
int pmhd_gpu_exchange(pmhd_mesh* mesh);

/* compute_dt of the current state (active cells). */
int pmhd_gpu_new_dt(pmhd_mesh* mesh, double* dt_out, pmhd_status* st);

/* One VL2 stage: stage 1 advances a copy of (u,b) by dt/2 with
 * donor-cell states; stage 2 advances the t^n state by dt with PLM states of
 * the half state.  Includes the trailing ghost exchange of the result.  After
 * stage 2, *dt_next (may be NULL) holds compute_dt of the new state. */
int pmhd_gpu_stage(pmhd_mesh* mesh, int stage, double dt, double* dt_next, pmhd_status* st);

/* vl2_step = stage 1 + stage 2. */
int pmhd_gpu_vl2_step(pmhd_mesh* mesh, double dt, double* dt_next, pmhd_status* st);

/* cmd_run inner loop: up to ncycles cycles or until
 * *t reaches tlim (dt capped to land exactly on tlim), starting
 * from *dt (pass <= 0 to compute it).  Updates *t, *dt, *cycles_done. */
int pmhd_gpu_run(pmhd_mesh* mesh, int ncycles, double tlim, double* t, double* dt,
                 int* cycles_done, pmhd_status* st);

/* ---- Multi-rank pieces (one process per GPU) -------------
 * A rank owns a subset of the blocks (gids at mesh creation).  A stage is then
 * pmhd_gpu_stage_compute + for dir in x1..x3 { pmhd_gpu_exchange_dir (blocks
 * with local neighbours) + halo pack -> transport -> unpack for the faces with
 * remote neighbours }, which reproduces exchange_ghosts' sequential sweeps
 * exactly.  half = 1 selects u^{n+1/2} (after stage 1), 0 the
 * current state (after stage 2).  Halo buffers are DEVICE pointers; message
 * layout = pack_boundary: variable-major (u0..u4, b1f, b2f,
 * b3f), each slab in k-j-i order.  pack/unpack return after the copy is done. */
int pmhd_gpu_stage_compute(pmhd_mesh* mesh, int stage, double dt, double* dt_next, pmhd_status* st);
/* Optional, between stage_compute(1) and the halo exchange that follows it:
 * enqueue stage 2's flux work on the tiles that read no ghost data (on a
 * second stream, after stage 1), so it runs while the halo is exchanged;
 * stage_compute(2, same dt) then does the remaining tiles.  "Overlapped with
 * interior updates" (north_star); a no-op where it does not apply
 * (profiling, split kernels, PMHD_OVERLAP=0).  vl2_step does this itself. */
int pmhd_gpu_stage_prefetch(pmhd_mesh* mesh, int stage, double dt);
int pmhd_gpu_exchange_dir(pmhd_mesh* mesh, int dir, int half);
/* doubles in the message that block side `side` (0 lower, 1 upper) receives */
int pmhd_gpu_halo_count(const pmhd_mesh* mesh, int dir, int side, long long* n);
/* slab block gid sends to its neighbour on `side` */
int pmhd_gpu_halo_pack(pmhd_mesh* mesh, int gid, int dir, int side, int half, double* dev_buf);
/* ghosts of block gid on `side`, from the neighbour's pack(..., 1 - side) */
int pmhd_gpu_halo_unpack(pmhd_mesh* mesh, int gid, int dir, int side, int half, const double* dev_buf);
/* Peer-memory halo (one node, NVLink / NVSwitch): instead of pack -> transport
 * -> unpack, pmhd_gpu_exchange_dir reads a remote neighbour's boundary
 * layers straight from its memory.  Every rank exports its state slab
 * (pmhd_gpu_slab: base + CUDA IPC handle, 64 bytes), maps the others'
 * (pmhd_gpu_ipc_open) and calls pmhd_gpu_peer_attach with the owner of every
 * gid and each rank's mapped base (NULL: no mapping, that rank's faces keep
 * using halo pack / unpack; a rank's own entry is ignored).  Ranks must have
 * created their meshes with their gids in ascending order.  Ordering is the
 * caller's: before exchange_dir(d) on any rank, every rank must have finished
 * the stage (d = x1) or its exchange_dir(d-1) -- a barrier per direction
 * (DistributedVL2 uses a stream-ordered NCCL all-reduce of one int). */
int pmhd_gpu_slab(const pmhd_mesh* mesh, void** base, void* ipc_handle /* 64 bytes or NULL */);
int pmhd_gpu_ipc_open(pmhd_ctx* ctx, const void* ipc_handle, void** base);
int pmhd_gpu_ipc_close(pmhd_ctx* ctx, void* base);
int pmhd_gpu_peer_attach(pmhd_mesh* mesh, int nranks, const int* owner_of_gid, void* const* rank_base);

/* Stream-ordered multi-rank mode (on != 0): exchange_dir / halo_pack /
 * halo_unpack return as soon as their kernels are enqueued on
 * pmhd_gpu_stream(ctx), and stage_compute(1) returns without synchronizing
 * (its floor count / error cell are reported by the following
 * stage_compute(2), whose status covers both stages).  The transport must
 * order its device work on that stream (e.g. NCCL issued on it).  Off
 * (default): every call returns once its results are complete. */
int pmhd_gpu_set_async(pmhd_mesh* mesh, int on);

/* Turbulence driving (definition in pmhd_host.h).  One
 * event = three calls; the caller combines the per-block partial sums over
 * all blocks in gid order (across ranks too), so every decomposition and the
 * CPU oracle form the same bits:
 *  1 drive_begin: nmode modes (k: nmode x 3 ints, c / s: nmode x 3 doubles)
 *    and the per-axis phase tables (host pointers, 5 x nx[a] doubles each);
 *    forms dv on every active cell and returns sums[4 b + q] =
 *    (sum rho, sum rho dv_x, sum rho dv_y, sum rho dv_z) of local block b,
 *    each (k, j) row summed over i, rows in (k, j) order;
 *  2 drive_energy(mean): dv' = dv - mean; sums[4 b + q] =
 *    (sum 1/2 rho |dv'|^2, sum m.dv', 0, 0);
 *  3 drive_apply(mean, s): m += (s rho) dv', E += KE(m_new) - KE(m), then the
 *    ghost exchange of blocks with local neighbours (multi-rank callers
 *    exchange the rest). */
int pmhd_gpu_drive_begin(pmhd_mesh* mesh, int nmode, const int* k, const double* c, const double* s,
                         const double* const* cos_tab, const double* const* sin_tab, double* sums);
int pmhd_gpu_drive_energy(pmhd_mesh* mesh, const double* mean, double* sums);
int pmhd_gpu_drive_apply(pmhd_mesh* mesh, const double* mean, double scale);

/* Diagnostics (PMHD_DIAG_*). */
int pmhd_gpu_diag(pmhd_mesh* mesh, int kind, double* out);

/* Region profiling (with_region, profiler.hpp:90-103; SPEC.md:527 names).
 * on = 1: every stage records CUDA events between its kernel groups,
 * launches the instrumented kernel instantiations (clock64 phase shares split
 * the fused kernels' times into the SPEC regions) and synchronizes at its
 * end.  on = 2: the same events around the product kernels, without the
 * phase instrumentation: riemann_ms then holds the whole flux-kernel time
 * and integrate_ms the whole update-kernel time (c2p / reconstruct / ct_emf
 * stay 0 for the fused kernels).  0 (default) adds no synchronization. */
int pmhd_gpu_set_profiling(pmhd_mesh* mesh, int on);
/* Accumulated region times (out may be NULL); reset != 0 zeroes them. */
int pmhd_gpu_region_times(pmhd_mesh* mesh, pmhd_region_times* out, int reset);

/* The context's CUDA stream (cudaStream_t) for interop: callers may record
 * events on it to time ABI calls.  Work a call forks to the context's
 * internal streams (the x2 flux launch beside x1 -> x3, host<->device
 * copies, a stage prefetch) joins back to it before the call returns, with
 * one exception: pmhd_gpu_vl2_step may leave its last x2 / x3 ghost
 * exchanges running beside the stream (they overlap the next step's x1
 * flux launch; PMHD_EARLY_X1=0 disables).  Every entry point that touches
 * the state orders itself after them; an event meant to close a timed
 * region of steps should be recorded after a device synchronize. */
void* pmhd_gpu_stream(const pmhd_ctx* ctx);

/* Name of the kernel variant compiled into this library ("fused", "split"...). */
const char* pmhd_gpu_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* PMHD_GPU_H_ */
