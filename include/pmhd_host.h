/*
 * pmhd_host.h -- C API of the host-side C++ library (libpmhd_host.so):
 * input-file parsing, MeshConfig/MeshBlock geometry and the problem
 * generators.  This is the host layer that sits above the GPU C-ABI
 * (pmhd_gpu.h); the reference defines it in
 *   parse_config
 *   MeshConfig/build_mesh
 *   init_linear_wave    SPEC.md:218-226   (WaveSetup SPEC.md:126-129)
 *   l1_error
 * plus the Orszag-Tang, blast and turbulence generators that BASELINE.json's
 * configs require (definitions in DESIGN.md / SURVEY.md §8d).
 */
#ifndef PMHD_HOST_H_
#define PMHD_HOST_H_

#include <stdint.h>

#include "pmhd_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PMHD_PGEN_LINEAR_WAVE = 0,
  PMHD_PGEN_ORSZAG_TANG = 1,
  PMHD_PGEN_BLAST = 2,
  PMHD_PGEN_TURBULENCE = 3,
  PMHD_PGEN_UNIFORM = 4
};

/* Linear-wave eigenmodes, ordered by eigenvalue (Athena++ wave_flag order):
 * 0 fast-left, 1 Alfven-left, 2 slow-left, 3 entropy, 4 slow-right,
 * 5 Alfven-right, 6 fast-right. */

/* RunConfig. */
typedef struct pmhd_run_config {
  pmhd_mesh_desc mesh;
  int pgen;                 /* PMHD_PGEN_*                                      */
  /* WaveSetup; background in the wave frame (n,t1,t2)    */
  double wave_amp;          /* A, default 1e-6                                  */
  int wave_n[3];            /* integer periods per domain, default (1,0,0)     */
  int wave_mode;            /* 0..6, default 6 (fast, right-going)              */
  double wave_rho, wave_p;  /* default 1, 0.6                                   */
  double wave_v[3];         /* (vn, vt1, vt2), default 0                        */
  double wave_b[3];         /* (bn, bt1, bt2), default (1, sqrt 2, 0.5)         */
  /* blast */
  double blast_pin, blast_pout, blast_r, blast_rho;
  double blast_b[3];
  /* turbulence */
  double turb_mach;
  uint64_t turb_seed;
  /* uniform state (pgen uniform): rho, v1..3, p, B1..3 */
  double uniform_w[8];
  /* run control */
  int nlim;                 /* cycle limit (-1: none)                           */
  double tlim;              /* time limit (<= 0: one wave period / pgen default) */
  int workers;              /* CPU workers (oracle / baseline)                  */
  int gpus;
  /* turbulence driving (BASELINE config 5 "driven"):
   * every turb_every cycles, a solenoidal velocity impulse injecting
   * turb_dedt x (time since the last event) of kinetic energy */
  int turb_drive;           /* 0: decaying (default), 1: driven                 */
  double turb_dedt;         /* energy injection rate, default 1                 */
  int turb_every;           /* cycles between driving events, default 1         */
} pmhd_run_config;

/* Defaults (empty text -> 16^3, one block). */
void pmhd_host_config_defaults(pmhd_run_config* cfg);

/* parse_config: "key = value" lines, '#' comments, later
 * keys override, unknown key or malformed value -> PMHD_ERR_INPUT with
 * *err_line set (1-based) and a message in err (may be NULL). */
int pmhd_host_config_parse(const char* text, pmhd_run_config* cfg, int* err_line, char* err,
                           int errlen);

/* MeshConfig invariants -> PMHD_ERR_CONFIG. */
int pmhd_host_validate(const pmhd_run_config* cfg, char* err, int errlen);

/* Block geometry: number of blocks, array extents (with ghosts), cell sizes. */
int pmhd_host_nblocks(const pmhd_run_config* cfg);
void pmhd_host_block_dims(const pmhd_run_config* cfg, int n[3]);
void pmhd_host_block_coords(const pmhd_run_config* cfg, int gid, int c[3]);

/* Problem generator: fills the ACTIVE cells and faces of block gid (ghosts are
 * left untouched; call exchange afterwards).  u: 8 vars (Bcc from the face
 * average), faces as in pmhd_gpu.h. */
int pmhd_host_pgen_block(const pmhd_run_config* cfg, int gid, double* u, double* b1f,
                         double* b2f, double* b3f);

/* Exact linear-wave solution at time t at the cell centres of the active
 * cells of block gid: 8 vars (rho, m1, m2, m3, E, B1, B2, B3), NCONS x n3 x
 * n2 x n1 layout (ghost entries untouched). */
int pmhd_host_exact_block(const pmhd_run_config* cfg, int gid, double t, double* u);

/* Linear-wave eigen data: eigenvalue (phase speed along n) of the selected
 * mode, right eigenvector (7 conserved wave-frame components), and the
 * residual ||(J - lambda I) r||_inf of the complex-step flux Jacobian. */
int pmhd_host_wave_eigen(const pmhd_run_config* cfg, double* lambda, double r[7],
                         double* residual);

/* Default end time of the problem (one wave period for linear waves). */
double pmhd_host_default_tlim(const pmhd_run_config* cfg);

/* PMHD1 snapshot: ASCII header lines "PMHD1", "dims n1 n2 n3",
 * "gamma g", "time t", "END", then little-endian fp64: the 8 conserved
 * variables over the GLOBAL active grid (variable-major, k-j-i), then the
 * global staggered b1f, b2f, b3f.  u/b*f[g] are the host arrays of block g
 * (layout of pmhd_gpu.h).  write: all blocks; read: fills the active cells
 * and faces of every block (ghosts untouched; exchange afterwards) and checks
 * dims / gamma -> PMHD_ERR_INPUT on mismatch or a malformed file. */
int pmhd_host_snapshot_write(const char* path, const pmhd_run_config* cfg, double t,
                             double* const* u, double* const* b1f, double* const* b2f,
                             double* const* b3f);
int pmhd_host_snapshot_read(const char* path, const pmhd_run_config* cfg, double* t, double* const* u,
                            double* const* b1f, double* const* b2f, double* const* b3f);

/* ---- Turbulence driving ---------------------------------
 * Impulsive solenoidal forcing: event e draws Fourier modes with integer
 * wavevectors 1 <= |k|^2 <= 4 (half space) from mt19937_64(turb_seed ^
 * (e+1) * golden) in the fixed (kx,ky,kz) loop order of the turbulence pgen;
 * dv(x) = sum_m c_m cos(2 pi k.x/L) + s_m sin(2 pi k.x/L), c_m and s_m
 * projected perpendicular to k.  cos/sin are products of per-axis tables
 * (k = -2..2 at the global cell centres), so every backend forms the same
 * bits. */
#define PMHD_DRIVE_MAX_MODES 64
typedef struct pmhd_drive_modes {
  int n;
  int k[PMHD_DRIVE_MAX_MODES][3];
  double c[PMHD_DRIVE_MAX_MODES][3];
  double s[PMHD_DRIVE_MAX_MODES][3];
} pmhd_drive_modes;
int pmhd_host_drive_modes(const pmhd_run_config* cfg, long long event, pmhd_drive_modes* out);
/* axis table: cos_tab[(k+2)*nx + g], sin_tab[...] for k = -2..2 and the
 * global cell index g in [0, nx[axis]) */
int pmhd_host_drive_tables(const pmhd_run_config* cfg, int axis, double* cos_tab, double* sin_tab);
/* impulse amplitude s >= 0 with a s^2 + b s = de (a = sum 1/2 rho |dv'|^2,
 * b = sum rho v.dv'): s = (-b + sqrt(b^2 + 4 a de)) / (2 a) */
double pmhd_host_drive_scale(double a, double b, double de);

/* ---- perf_model: roofline (Eq. 1), architectural
 * efficiency (Eq. 2), performance-portability metric (Eq. 3) over platform
 * records (Table 2 schema).  Pure functions; bandwidths in B/s, peaks in
 * FLOP/s. */
#define PMHD_PERF_MAX_SPACES 8
typedef struct pmhd_platform {
  char id[32];
  double t_peak;                                /* FLOP/s (double precision) */
  int nspace;
  char space[PMHD_PERF_MAX_SPACES][16];         /* memory-space labels ("dram", "l2", ...) */
  double bw[PMHD_PERF_MAX_SPACES];              /* B/s per space */
} pmhd_platform;

/* load_platform_table: CSV text with header `id,t_peak_gflops,bw_<space>_gbs...`
 * (GFLOP/s, GB/s).  Missing / non-numeric / non-positive field ->
 * PMHD_ERR_INPUT with the 1-based line in *err_line.  Empty text -> 0 rows. */
int pmhd_perf_load_platforms(const char* text, pmhd_platform* out, int max_rows, int* n_rows,
                             int* err_line, char* err, int errlen);
/* The same schema back (round trip of load); returns the bytes needed. */
int pmhd_perf_format_platforms(const pmhd_platform* p, int n, char* buf, int buflen);
/* roofline_cap (Eq. 1) for one kernel intensity set: P_max = min over the
 * given spaces of min(T_peak, B(space) * I(space)); *binding = -1 when the
 * compute peak binds, else the index of the binding space.  Unknown space ->
 * PMHD_ERR_INPUT. */
int pmhd_perf_roofline_cap(const pmhd_platform* p, const char* const* spaces, const double* intensity,
                           int n, double* cap, int* binding);
/* arch_efficiency (Eq. 2): e = eps / cap; *flag = 1 when e > 1 (reported, not
 * clamped).  cap <= 0 -> PMHD_ERR_INPUT. */
int pmhd_perf_arch_efficiency(double eps, double cap, double* e, int* flag);
/* pp_metric (Eq. 3): |H| / sum 1/e over the platforms, 0 if any platform is
 * unsupported (supported[i] == 0); a supported e <= 0 -> PMHD_ERR_INPUT. */
int pmhd_perf_pp_metric(const double* e, const int* supported, int n, double* P);

#ifdef __cplusplus
}
#endif

#endif /* PMHD_HOST_H_ */
