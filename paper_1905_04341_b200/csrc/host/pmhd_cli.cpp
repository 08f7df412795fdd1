// pmhd_cli.cpp -- the reference's command-line front end (bench_cli,
// SPEC.md:445-513) for the GPU path: C++ host code over the two C ABIs
// (pmhd_host.h: input files + problem generators; pmhd_gpu.h: the solver).
//
//   pmhd run   --config <file> [--out <dir>] [--device <d>] [--restart <snapshot>]
//                                                             (cmd_run)
//   pmhd bench --config <file> [--cycles <n>] [--warmup <w>]  (cmd_bench)
//   pmhd report --config <file> [--cycles <n>] [--warmup <w>] [--falg <csv>] [--out <dir>]
//        Fig. 3 analogue (with_region report): profile.csv =
//        region, calls, time_s, time_normalized, flops, bytes, intensity
//   pmhd roofline --config <file> --platform <csv> [--platform-id <id>] [--falg <csv>] ...
//        cmd_roofline: Eq. 1-3 reports roofline.csv and
//        portability.csv (perf_model)
//
// run: evolves to tlim (default: one wave period) or nlim cycles, prints
// cycles / wall time / cell-updates per second, writes errors.csv (linear
// wave L1 errors) and a PMHD1 snapshot.  Solver
// errors exit non-zero.
#include <sys/stat.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "pmhd_gpu.h"
#include "pmhd_host.h"

namespace {

struct Args {
  std::string cmd, config, out = ".", restart, falg = "profiles/falg_regions.csv", platform,
      platform_id = "b200";
  int device = 0, cycles = 10, warmup = 2;
};

int usage() {
  std::fprintf(stderr,
               "usage: pmhd run|bench|report|roofline --config <file> [--out <dir>] [--device <d>] "
               "[--cycles <n>] [--warmup <w>] [--restart <snapshot>] [--falg <csv>] "
               "[--platform <csv>] [--platform-id <id>]\n");
  return 2;
}

std::string slurp(const std::string& path) {
  std::ifstream f(path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

struct Blocks {
  int n[3];
  size_t nc, n1f, n2f, n3f;
  std::vector<std::vector<double>> u, b1, b2, b3;
  void alloc(int nb, const int dims[3]) {
    for (int a = 0; a < 3; ++a) n[a] = dims[a];
    nc = size_t(n[0]) * n[1] * n[2];
    n1f = size_t(n[0] + 1) * n[1] * n[2];
    n2f = size_t(n[0]) * (n[1] + 1) * n[2];
    n3f = size_t(n[0]) * n[1] * (n[2] + 1);
    u.assign(nb, std::vector<double>(8 * nc));
    b1.assign(nb, std::vector<double>(n1f));
    b2.assign(nb, std::vector<double>(n2f));
    b3.assign(nb, std::vector<double>(n3f));
  }
};

// Turbulence driving: the host side of one forcing event
// over the drive_* ABI; sums combined over blocks in gid order.
struct Drive {
  const pmhd_run_config* cfg = nullptr;
  std::vector<double> ct[3], st[3];
  long long event = 0;
  double since = 0.0;  // time since the last event
  void init(const pmhd_run_config& c) {
    cfg = &c;
    for (int a = 0; a < 3; ++a) {
      ct[a].assign(5 * size_t(c.mesh.nx[a]), 0.0);
      st[a].assign(5 * size_t(c.mesh.nx[a]), 0.0);
      pmhd_host_drive_tables(&c, a, ct[a].data(), st[a].data());
    }
  }
  int kick(pmhd_mesh* mesh, int nb) {
    pmhd_drive_modes md;
    pmhd_host_drive_modes(cfg, event, &md);
    std::vector<int> k(3 * md.n);
    std::vector<double> c(3 * md.n), s(3 * md.n), sums(4 * size_t(nb));
    for (int m = 0; m < md.n; ++m)
      for (int a = 0; a < 3; ++a) {
        k[3 * m + a] = md.k[m][a];
        c[3 * m + a] = md.c[m][a];
        s[3 * m + a] = md.s[m][a];
      }
    const double* cp[3] = {ct[0].data(), ct[1].data(), ct[2].data()};
    const double* sp[3] = {st[0].data(), st[1].data(), st[2].data()};
    int rc = pmhd_gpu_drive_begin(mesh, md.n, k.data(), c.data(), s.data(), cp, sp, sums.data());
    if (rc) return rc;
    double tot[4] = {0.0, 0.0, 0.0, 0.0};
    for (int b = 0; b < nb; ++b)
      for (int q = 0; q < 4; ++q) tot[q] = tot[q] + sums[4 * b + q];
    const double mean[3] = {tot[1] / tot[0], tot[2] / tot[0], tot[3] / tot[0]};
    rc = pmhd_gpu_drive_energy(mesh, mean, sums.data());
    if (rc) return rc;
    double te[2] = {0.0, 0.0};
    for (int b = 0; b < nb; ++b)
      for (int q = 0; q < 2; ++q) te[q] = te[q] + sums[4 * b + q];
    const double cells = double(cfg->mesh.nx[0]) * cfg->mesh.nx[1] * cfg->mesh.nx[2];
    const double scale = pmhd_host_drive_scale(te[0], te[1], cfg->turb_dedt * since * cells);
    rc = pmhd_gpu_drive_apply(mesh, mean, scale);
    ++event;
    since = 0.0;
    return rc;
  }
};

// cmd_run / cmd_bench cycle loop; with turb_drive, chunks of turb_every
// cycles separated by forcing events (dt recomputed after each).
int run_cycles(pmhd_mesh* mesh, const pmhd_run_config& cfg, Drive* drv, int nb, int ncycles, double tlim,
               double* t, double* dt, int* done, pmhd_status* st) {
  if (!cfg.turb_drive) return pmhd_gpu_run(mesh, ncycles, tlim, t, dt, done, st);
  *done = 0;
  while ((ncycles < 0 || *done < ncycles) && (tlim <= 0.0 || *t < tlim)) {
    int chunk = cfg.turb_every;
    if (ncycles >= 0) chunk = std::min(chunk, ncycles - *done);
    const double t0 = *t;
    int d = 0;
    const int rc = pmhd_gpu_run(mesh, chunk, tlim, t, dt, &d, st);
    if (rc) return rc;
    *done += d;
    drv->since += *t - t0;
    if (d < chunk || d == 0) break;  // reached tlim
    if (drv->kick(mesh, nb)) return PMHD_ERR_CUDA;
    *dt = 0.0;  // recompute after the kick
  }
  return PMHD_OK;
}

// Algorithmic flops per cell-update by region (tools/count_falg.py: the CPU
// oracle on the CountingScalar restatement, one cycle of the bench config).
bool load_falg(const std::string& path, std::vector<std::pair<std::string, double>>* rows) {
  std::ifstream f(path);
  if (!f) return false;
  std::string line;
  std::getline(f, line);  // header region,flops_per_cell_update
  while (std::getline(f, line)) {
    const size_t c = line.find(',');
    if (c == std::string::npos) continue;
    rows->push_back({line.substr(0, c), std::atof(line.c_str() + c + 1)});
  }
  return !rows->empty();
}

// Streaming-byte model of THIS implementation's kernels per cell-update
// (8 B per array element read or written once per kernel, SPEC.md:330's
// convention applied to the fused kernels; 3D, both stages): the flux kernels
// read the 8 state arrays over their stencil tiles (~1.15 cells per face) and
// write 8 face arrays per direction (+3 cell-E arrays in the last direction);
// the update kernel reads 9 EMF inputs + 3 cell-E (ct_emf) and 15 fluxes + 8
// base state, writing 8 (integrate).  Loads are attributed to c2p and stores
// to riemann (reconstruct works in shared memory).
double region_bytes(const std::string& r, int dim) {
  const double nd = dim;
  if (r == "c2p") return 2.0 * nd * 8.0 * 1.15 * 8.0;
  if (r == "riemann") return 2.0 * (nd * 8.0 + 3.0) * 8.0;
  if (r == "ct_emf") return 2.0 * (3.0 * nd + 3.0) * 8.0;
  if (r == "integrate") return 2.0 * (5.0 * nd + 16.0) * 8.0;
  return 0.0;
}

int cmd_report(const Args& a, const pmhd_run_config& cfg, pmhd_mesh* mesh, long long cells, double* t,
               double* dt) {
  std::vector<std::pair<std::string, double>> falg;
  if (!load_falg(a.falg, &falg)) {
    std::fprintf(stderr, "no flop table %s (python tools/count_falg.py writes it)\n", a.falg.c_str());
    return 1;
  }
  pmhd_status st;
  int done = 0;
  if (pmhd_gpu_run(mesh, a.warmup, -1.0, t, dt, &done, &st)) return 1;
  // timed pass (no profiling: no region synchronisation) for epsilon
  auto t0 = std::chrono::steady_clock::now();
  if (pmhd_gpu_run(mesh, a.cycles, -1.0, t, dt, &done, &st)) return 1;
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  // profiled pass for the region breakdown
  pmhd_region_times rt;
  pmhd_gpu_region_times(mesh, nullptr, 1);
  pmhd_gpu_set_profiling(mesh, 1);
  auto tp = std::chrono::steady_clock::now();
  if (pmhd_gpu_run(mesh, a.cycles, -1.0, t, dt, &done, &st)) return 1;
  const double wall_prof = std::chrono::duration<double>(std::chrono::steady_clock::now() - tp).count();
  pmhd_gpu_set_profiling(mesh, 0);
  pmhd_gpu_region_times(mesh, &rt, 1);
  const int ncyc = done;
  const double upd = double(cells) * ncyc;
  struct Reg { std::string name; double ms; };
  const std::vector<Reg> regs = {{"c2p", rt.c2p_ms},         {"reconstruct", rt.reconstruct_ms},
                                 {"riemann", rt.riemann_ms}, {"ct_emf", rt.ct_emf_ms},
                                 {"integrate", rt.integrate_ms}, {"boundary", rt.boundary_ms}};
  double fl_tot = 0.0;
  for (auto& f : falg) fl_tot += f.second;
  mkdir(a.out.c_str(), 0755);
  const int dim = cfg.mesh.nx[2] > 1 ? 3 : 2;
  if (a.cmd == "report") {
    const double rie = rt.riemann_ms > 0 ? rt.riemann_ms : 1.0;
    FILE* f = std::fopen((a.out + "/profile.csv").c_str(), "w");
    std::fprintf(f, "region,calls,time_s,time_normalized,flops,bytes,intensity\n");
    double tot_ms = 0.0;
    for (auto& r : regs) {
      double fpc = 0.0;
      for (auto& q : falg) if (q.first == r.name || (r.name == "integrate" && q.first == "dt")) fpc += q.second;
      const double flops = fpc * upd, bytes = region_bytes(r.name, dim) * upd;
      std::fprintf(f, "%s,%lld,%.9g,%.6g,%.6g,%.6g,%.6g\n", r.name.c_str(), (long long)rt.calls,
                   r.ms * 1e-3, r.ms / rie, flops, bytes, bytes > 0 ? flops / bytes : 0.0);
      tot_ms += r.ms;
    }
    std::fclose(f);
    // SPEC.md:546 (acceptance 11): named regions partition >= 90 % of a cycle
    std::printf("profile.csv: %d cycles; regions cover %.1f %% of the profiled wall time (%.3f of %.3f ms); "
                "unprofiled pass %.4e cell-updates/s\n",
                ncyc, 100.0 * tot_ms / (wall_prof * 1e3), tot_ms, wall_prof * 1e3, upd / wall);
    return 0;
  }
  // cmd_roofline: epsilon from the timed pass, intensity from F_alg / B_alg
  std::ifstream pf(a.platform);
  std::stringstream ss;
  ss << pf.rdbuf();
  pmhd_platform plats[16];
  int np = 0, line = 0;
  char err[256];
  if (!pf || pmhd_perf_load_platforms(ss.str().c_str(), plats, 16, &np, &line, err, sizeof(err))) {
    std::fprintf(stderr, "platform file %s: line %d: %s\n", a.platform.c_str(), line, err);
    return 1;
  }
  int host = -1;
  for (int i = 0; i < np; ++i) if (a.platform_id == plats[i].id) host = i;
  if (host < 0) {
    std::fprintf(stderr, "no platform record '%s' in %s\n", a.platform_id.c_str(), a.platform.c_str());
    return 1;
  }
  const double b_alg = 320.0;  // compulsory bytes per cell-update
  const double eps = fl_tot * upd / wall;
  const double I = fl_tot / b_alg;
  const char* sp = "dram";
  double cap = 0.0, e = 0.0;
  int bind = 0, flag = 0;
  if (pmhd_perf_roofline_cap(&plats[host], &sp, &I, 1, &cap, &bind) ||
      pmhd_perf_arch_efficiency(eps, cap, &e, &flag)) {
    std::fprintf(stderr, "platform '%s' has no dram bandwidth\n", a.platform_id.c_str());
    return 1;
  }
  FILE* f = std::fopen((a.out + "/portability.csv").c_str(), "w");
  std::fprintf(f, "platform,space,epsilon_gflops,cap_gflops,efficiency\n");
  std::fprintf(f, "%s,%s,%.6f,%.6f,%.6f\n", plats[host].id, sp, eps / 1e9, cap / 1e9, e);
  double P = 0.0;
  pmhd_perf_pp_metric(&e, nullptr, 1, &P);
  std::fprintf(f, "pp_metric_%s,%.6f\n", sp, P);
  std::fclose(f);
  f = std::fopen((a.out + "/roofline.csv").c_str(), "w");  // Fig. 4-style sample points
  std::fprintf(f, "series,space,intensity,gflops\n");
  for (int q = 0; q <= 48; ++q) {
    const double x = std::pow(2.0, -8.0 + q * 0.5);
    double c;
    int b;
    pmhd_perf_roofline_cap(&plats[host], &sp, &x, 1, &c, &b);
    std::fprintf(f, "ceiling,%s,%.6g,%.6f\n", sp, x, c / 1e9);
  }
  std::fprintf(f, "achieved,%s,%.6g,%.6f\n", sp, I, eps / 1e9);
  std::fclose(f);
  std::printf("roofline: eps %.1f GFLOP/s at I = %.3f flop/B, cap %.1f GFLOP/s (%s-bound), e = %.4f%s\n",
              eps / 1e9, I, cap / 1e9, bind < 0 ? "compute" : sp, e, flag ? " (>1: model inconsistency)" : "");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  // Load every kernel of libpmhd_gpu.so when the context is created rather
  // than at its first launch: with lazy loading `run` would time the loading
  // of each kernel inside its first cycle (~10 ms, 8 % of the 64^3 wave's
  // 0.1 s run).  A CUDA_MODULE_LOADING the user set is kept.
  setenv("CUDA_MODULE_LOADING", "EAGER", 0);
  Args a;
  if (argc < 2) return usage();
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    auto next = [&]() { return (i + 1 < argc) ? std::string(argv[++i]) : std::string(); };
    if (s == "--config") a.config = next();
    else if (s == "--out") a.out = next();
    else if (s == "--restart") a.restart = next();
    else if (s == "--device") a.device = std::atoi(next().c_str());
    else if (s == "--cycles") a.cycles = std::atoi(next().c_str());
    else if (s == "--warmup") a.warmup = std::atoi(next().c_str());
    else if (s == "--falg") a.falg = next();
    else if (s == "--platform") a.platform = next();
    else if (s == "--platform-id") a.platform_id = next();
    else return usage();
  }
  if ((a.cmd != "run" && a.cmd != "bench" && a.cmd != "report" && a.cmd != "roofline") || a.config.empty())
    return usage();
  if (a.cmd == "roofline" && a.platform.empty()) return usage();

  pmhd_run_config cfg;
  pmhd_host_config_defaults(&cfg);
  int line = 0;
  char err[256];
  if (pmhd_host_config_parse(slurp(a.config).c_str(), &cfg, &line, err, sizeof(err)) != PMHD_OK) {
    std::fprintf(stderr, "parse error: %s\n", err);
    return 1;
  }
  if (pmhd_host_validate(&cfg, err, sizeof(err)) != PMHD_OK) {
    std::fprintf(stderr, "config error: %s\n", err);
    return 1;
  }
  pmhd_ctx* ctx = nullptr;
  if (pmhd_gpu_ctx_create(a.device, &ctx) != PMHD_OK) {
    std::fprintf(stderr, "no usable sm_100 device %d (there is no CPU fallback)\n", a.device);
    return 1;
  }
  pmhd_mesh* mesh = nullptr;
  if (pmhd_gpu_mesh_create(ctx, &cfg.mesh, nullptr, 0, &mesh) != PMHD_OK) {
    std::fprintf(stderr, "mesh: %s\n", pmhd_gpu_last_error(ctx));
    return 1;
  }
  const int nb = pmhd_host_nblocks(&cfg);
  int dims[3];
  pmhd_host_block_dims(&cfg, dims);
  Blocks B;
  B.alloc(nb, dims);
  std::vector<double*> pu(nb), p1(nb), p2(nb), p3(nb);
  for (int g = 0; g < nb; ++g) {
    pu[g] = B.u[g].data(); p1[g] = B.b1[g].data(); p2[g] = B.b2[g].data(); p3[g] = B.b3[g].data();
  }
  double t = 0.0, dt = 0.0;
  if (!a.restart.empty()) {  // restart from a PMHD1 snapshot
    if (pmhd_host_snapshot_read(a.restart.c_str(), &cfg, &t, pu.data(), p1.data(), p2.data(),
                                p3.data()) != PMHD_OK) {
      std::fprintf(stderr, "restart: %s is not a PMHD1 snapshot of this mesh\n", a.restart.c_str());
      return 1;
    }
  } else {
    for (int g = 0; g < nb; ++g) pmhd_host_pgen_block(&cfg, g, pu[g], p1[g], p2[g], p3[g]);
  }
  for (int g = 0; g < nb; ++g) pmhd_gpu_upload_block(mesh, g, pu[g], p1[g], p2[g], p3[g]);
  pmhd_gpu_exchange(mesh);
  const long long cells = (long long)cfg.mesh.nx[0] * cfg.mesh.nx[1] * cfg.mesh.nx[2];
  pmhd_status st;
  int done = 0;
  Drive drv;
  if (cfg.turb_drive) drv.init(cfg);

  if (a.cmd == "bench") {
    // cmd_bench: warm-up cycles, then timed cycles; CSV row
    int rc = run_cycles(mesh, cfg, &drv, nb, a.warmup, -1.0, &t, &dt, &done, &st);
    auto t0 = std::chrono::steady_clock::now();
    if (!rc) rc = run_cycles(mesh, cfg, &drv, nb, a.cycles, -1.0, &t, &dt, &done, &st);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (rc) {
      std::fprintf(stderr, "solver error %d: %s\n", rc, pmhd_gpu_last_error(ctx));
      return 1;
    }
    std::printf("size,policy,workers,cycles,wall_s,cell_updates_per_s\n");
    std::printf("%dx%dx%d,gpu-%s,1,%d,%.6f,%.6e\n", cfg.mesh.nx[0], cfg.mesh.nx[1], cfg.mesh.nx[2],
                pmhd_gpu_build_info(), done, wall, double(cells) * done / wall);
    return 0;
  }

  if (a.cmd == "report" || a.cmd == "roofline") return cmd_report(a, cfg, mesh, cells, &t, &dt);

  // cmd_run
  const double tlim = pmhd_host_default_tlim(&cfg);
  auto t0 = std::chrono::steady_clock::now();
  int rc = run_cycles(mesh, cfg, &drv, nb, cfg.nlim, tlim, &t, &dt, &done, &st);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (rc == PMHD_ERR_UNPHYSICAL) {
    std::fprintf(stderr, "unphysical state in stage 'stage%d' at cell (k=%d, j=%d, i=%d)\n", st.stage,
                 st.k, st.j, st.i);
    return 1;
  }
  if (rc) {
    std::fprintf(stderr, "solver error %d: %s\n", rc, pmhd_gpu_last_error(ctx));
    return 1;
  }
  std::printf("cycles %d  time %.9g  wall %.3f s  cell-updates/s %.4e  floors %lld\n", done, t, wall,
              double(cells) * done / wall, st.floor_count);
  double divb = 0.0;
  pmhd_gpu_diag(mesh, PMHD_DIAG_DIVB_MAX, &divb);
  std::printf("max|div B| %.3e\n", divb);
  for (int g = 0; g < nb; ++g)
    pmhd_gpu_download_block(mesh, g, B.u[g].data(), nullptr, B.b1[g].data(), B.b2[g].data(),
                            B.b3[g].data());
  mkdir(a.out.c_str(), 0755);
  pmhd_host_snapshot_write((a.out + "/snapshot.pmhd").c_str(), &cfg, t, pu.data(), p1.data(), p2.data(),
                           p3.data());
  if (cfg.pgen == PMHD_PGEN_LINEAR_WAVE) {  // l1_error -> errors.csv
    std::vector<double> ex(8 * B.nc);
    double l1[8] = {0};
    const int ng = cfg.mesh.ng, g3 = cfg.mesh.nx[2] > 1 ? ng : 0;
    for (int g = 0; g < nb; ++g) {
      pmhd_host_exact_block(&cfg, g, t, ex.data());
      for (int v = 0; v < 8; ++v)
        for (int k = g3; k < g3 + cfg.mesh.mb[2]; ++k)
          for (int j = ng; j < ng + cfg.mesh.mb[1]; ++j)
            for (int i = ng; i < ng + cfg.mesh.mb[0]; ++i) {
              const size_t c = v * B.nc + (size_t(k) * B.n[1] + j) * B.n[0] + i;
              l1[v] += std::fabs(B.u[g][c] - ex[c]);
            }
    }
    double comb = 0.0;
    for (double& x : l1) { x /= double(cells); comb += x * x; }
    comb = std::sqrt(comb);
    FILE* f = std::fopen((a.out + "/errors.csv").c_str(), "w");
    std::fprintf(f, "resolution,cycles,L1_rho,L1_m1,L1_m2,L1_m3,L1_E,L1_B1,L1_B2,L1_B3,L1_combined\n");
    std::fprintf(f, "%d,%d", cfg.mesh.nx[0], done);
    for (double x : l1) std::fprintf(f, ",%.17g", x);
    std::fprintf(f, ",%.17g\n", comb);
    std::fclose(f);
    std::printf("L1 combined %.6e (errors.csv)\n", comb);
  }
  pmhd_gpu_mesh_destroy(mesh);
  pmhd_gpu_ctx_destroy(ctx);
  return 0;
}
