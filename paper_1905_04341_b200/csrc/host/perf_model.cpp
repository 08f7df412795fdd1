// perf_model.cpp -- the reference's perf_model module on
// the host: Eq. 1 roofline cap, Eq. 2 architectural efficiency, Eq. 3
// performance-portability metric, and the Table 2 platform CSV
// (load_platform_table).  Used by `pmhd roofline` / `pmhd report`.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "pmhd_gpu.h"
#include "pmhd_host.h"

namespace {

std::string trim(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && std::isspace(static_cast<unsigned char>(s[a]))) ++a;
  while (b > a && std::isspace(static_cast<unsigned char>(s[b - 1]))) --b;
  return s.substr(a, b - a);
}

std::vector<std::string> split_csv(const std::string& line) {
  std::vector<std::string> f;
  std::string cur;
  for (char c : line) {
    if (c == ',') { f.push_back(trim(cur)); cur.clear(); }
    else cur += c;
  }
  f.push_back(trim(cur));
  return f;
}

bool to_num(const std::string& s, double* v) {
  if (s.empty()) return false;
  char* end = nullptr;
  *v = std::strtod(s.c_str(), &end);
  return end && *end == '\0' && std::isfinite(*v);
}

int perr(int line, const std::string& msg, int* err_line, char* err, int errlen) {
  if (err_line) *err_line = line;
  if (err && errlen > 0) std::snprintf(err, errlen, "%s", msg.c_str());
  return PMHD_ERR_INPUT;
}

}  // namespace

extern "C" {

int pmhd_perf_load_platforms(const char* text, pmhd_platform* out, int max_rows, int* n_rows,
                             int* err_line, char* err, int errlen) {
  if (n_rows) *n_rows = 0;
  if (!text) return PMHD_OK;
  std::istringstream in(text);
  std::string line;
  int ln = 0, n = 0;
  std::vector<std::string> hdr;
  while (std::getline(in, line)) {
    ++ln;
    const std::string t = trim(line);
    if (t.empty() || t[0] == '#') continue;
    const std::vector<std::string> f = split_csv(t);
    if (hdr.empty()) {  // header
      if (f.size() < 2 || f[0] != "id" || f[1] != "t_peak_gflops")
        return perr(ln, "header must start with id,t_peak_gflops", err_line, err, errlen);
      if (f.size() - 2 > PMHD_PERF_MAX_SPACES) return perr(ln, "too many memory spaces", err_line, err, errlen);
      for (size_t c = 2; c < f.size(); ++c) {
        const std::string& h = f[c];
        if (h.size() < 8 || h.compare(0, 3, "bw_") != 0 || h.compare(h.size() - 4, 4, "_gbs") != 0 ||
            h.size() - 7 >= sizeof(out->space[0]))
          return perr(ln, "bandwidth column must be bw_<space>_gbs: " + h, err_line, err, errlen);
        for (size_t d = 2; d < c; ++d)
          if (f[d] == h) return perr(ln, "duplicate memory space " + h, err_line, err, errlen);
      }
      hdr = f;
      continue;
    }
    if (f.size() != hdr.size()) return perr(ln, "wrong number of fields", err_line, err, errlen);
    if (n >= max_rows) return perr(ln, "too many platforms", err_line, err, errlen);
    pmhd_platform p;
    std::memset(&p, 0, sizeof(p));
    if (f[0].empty() || f[0].size() >= sizeof(p.id)) return perr(ln, "bad platform id", err_line, err, errlen);
    std::snprintf(p.id, sizeof(p.id), "%s", f[0].c_str());
    double v;
    if (!to_num(f[1], &v) || !(v > 0.0)) return perr(ln, "t_peak_gflops must be a positive number", err_line, err, errlen);
    p.t_peak = v * 1e9;
    p.nspace = int(hdr.size()) - 2;
    for (int c = 0; c < p.nspace; ++c) {
      const std::string& h = hdr[c + 2];
      std::snprintf(p.space[c], sizeof(p.space[c]), "%s", h.substr(3, h.size() - 7).c_str());
      if (!to_num(f[c + 2], &v) || !(v > 0.0))
        return perr(ln, "bandwidth must be a positive number: " + h, err_line, err, errlen);
      p.bw[c] = v * 1e9;
    }
    out[n++] = p;
  }
  if (n_rows) *n_rows = n;
  return PMHD_OK;
}

int pmhd_perf_format_platforms(const pmhd_platform* p, int n, char* buf, int buflen) {
  std::string s;
  if (n > 0) {
    s = "id,t_peak_gflops";
    for (int c = 0; c < p[0].nspace; ++c) s += std::string(",bw_") + p[0].space[c] + "_gbs";
    s += "\n";
    char tmp[64];
    for (int r = 0; r < n; ++r) {
      s += p[r].id;
      std::snprintf(tmp, sizeof(tmp), ",%.17g", p[r].t_peak / 1e9);
      s += tmp;
      for (int c = 0; c < p[r].nspace; ++c) {
        std::snprintf(tmp, sizeof(tmp), ",%.17g", p[r].bw[c] / 1e9);
        s += tmp;
      }
      s += "\n";
    }
  }
  if (buf && buflen > 0) std::snprintf(buf, buflen, "%s", s.c_str());
  return int(s.size()) + 1;
}

int pmhd_perf_roofline_cap(const pmhd_platform* p, const char* const* spaces, const double* intensity,
                           int n, double* cap, int* binding) {
  if (!p || !cap || (n > 0 && (!spaces || !intensity))) return PMHD_ERR_INPUT;
  double best = p->t_peak;
  int bind = -1;
  for (int q = 0; q < n; ++q) {
    int c = -1;
    for (int s = 0; s < p->nspace; ++s)
      if (std::strcmp(p->space[s], spaces[q]) == 0) c = s;
    if (c < 0 || !(intensity[q] >= 0.0)) return PMHD_ERR_INPUT;
    const double lim = p->bw[c] * intensity[q];
    if (lim < best) { best = lim; bind = q; }
  }
  *cap = best;
  if (binding) *binding = bind;
  return PMHD_OK;
}

int pmhd_perf_arch_efficiency(double eps, double cap, double* e, int* flag) {
  if (!e || !(cap > 0.0) || !(eps >= 0.0)) return PMHD_ERR_INPUT;
  *e = eps / cap;
  if (flag) *flag = (*e > 1.0) ? 1 : 0;
  return PMHD_OK;
}

int pmhd_perf_pp_metric(const double* e, const int* supported, int n, double* P) {
  if (!P || n < 1 || !e) return PMHD_ERR_INPUT;
  for (int i = 0; i < n; ++i)
    if (supported && !supported[i]) { *P = 0.0; return PMHD_OK; }  // Eq. 3 "0 otherwise"
  // the reciprocals are summed in ascending order, so the result does not
  // depend on the order the platforms are listed in (permutation invariance)
  std::vector<double> r(n);
  for (int i = 0; i < n; ++i) {
    if (!(e[i] > 0.0)) return PMHD_ERR_INPUT;
    r[i] = 1.0 / e[i];
  }
  std::sort(r.begin(), r.end());
  double s = 0.0;
  for (double x : r) s += x;
  *P = double(n) / s;
  return PMHD_OK;
}

}  // extern "C"
