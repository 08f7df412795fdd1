// pmhd_cli.cpp -- the reference's command-line front end (bench_cli,
// SPEC.md:445-513) for the GPU path: C++ host code over the two C ABIs
// (pmhd_host.h: input files + problem generators; pmhd_gpu.h: the solver).
//
//   pmhd run   --config <file> [--out <dir>] [--device <d>] [--restart <snapshot>]
//                                                             (cmd_run)
//   pmhd bench --config <file> [--cycles <n>] [--warmup <w>]  (cmd_bench)
//
// run: evolves to tlim (default: one wave period) or nlim cycles, prints
// cycles / wall time / cell-updates per second, writes errors.csv (linear
// wave L1 errors) and a PMHD1 snapshot.  Solver
// errors exit non-zero.
#include <sys/stat.h>

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
  std::string cmd, config, out = ".", restart;
  int device = 0, cycles = 10, warmup = 2;
};

int usage() {
  std::fprintf(stderr,
               "usage: pmhd run|bench --config <file> [--out <dir>] [--device <d>] [--cycles <n>] "
               "[--warmup <w>] [--restart <snapshot>]\n");
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

}  // namespace

int main(int argc, char** argv) {
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
    else return usage();
  }
  if ((a.cmd != "run" && a.cmd != "bench") || a.config.empty()) return usage();

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

  if (a.cmd == "bench") {
    // cmd_bench: warm-up cycles, then timed cycles; CSV row
    int rc = pmhd_gpu_run(mesh, a.warmup, -1.0, &t, &dt, &done, &st);
    auto t0 = std::chrono::steady_clock::now();
    if (!rc) rc = pmhd_gpu_run(mesh, a.cycles, -1.0, &t, &dt, &done, &st);
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

  // cmd_run
  const double tlim = pmhd_host_default_tlim(&cfg);
  auto t0 = std::chrono::steady_clock::now();
  int rc = pmhd_gpu_run(mesh, cfg.nlim, tlim, &t, &dt, &done, &st);
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
