// oracle/counting.hpp -- TEST INFRASTRUCTURE (oracle), not product code.
//
// Restatement of the reference's flop-tallying scalar
//   /root/reference/proj/include/pmhd/exec/counting.hpp:31-96 (FlopCounts, CountingScalar)
// add/sub, mul, div and sqrt each count 1; a multiply followed by an add counts
// 2 (the FMA = 2 convention), which holds because the oracle is
// compiled with -ffp-contract=off (proj/CMakeLists.txt:11-14).  Unary minus,
// fabs, fmin/fmax, copysign and comparisons are free (counting.hpp:55,80-92).
// The tally is global and not thread-safe: counting runs use one worker
// (counting.hpp:17-18).
#ifndef ORACLE_COUNTING_HPP_
#define ORACLE_COUNTING_HPP_

#include <cmath>

namespace oracle {

struct FlopTally {
  double add = 0.0, mul = 0.0, div = 0.0, sqrt_n = 0.0;
  double total() const { return add + mul + div + sqrt_n; }
  void reset() { add = mul = div = sqrt_n = 0.0; }
};

inline FlopTally g_tally;
// Per-region split of the tally in the profiling-region names of SPEC.md:527
// ([0] c2p, [1] reconstruct, [2] riemann, [3] ct_emf, [4] integrate incl. CT
// face update and end-of-stage c2p; dt = the rest of a cycle), so each GPU
// kernel region gets its own algorithmic flops.  Only counting meshes (one
// worker) move the tally.
inline double g_region[5] = {0.0, 0.0, 0.0, 0.0, 0.0};

class Counting {
 public:
  Counting() = default;
  Counting(double v) : v_(v) {}  // NOLINT: implicit, literals appear in kernels
  double value() const { return v_; }

  Counting operator-() const { return Counting(-v_); }
  friend Counting operator+(Counting a, Counting b) { g_tally.add += 1; return Counting(a.v_ + b.v_); }
  friend Counting operator-(Counting a, Counting b) { g_tally.add += 1; return Counting(a.v_ - b.v_); }
  friend Counting operator*(Counting a, Counting b) { g_tally.mul += 1; return Counting(a.v_ * b.v_); }
  friend Counting operator/(Counting a, Counting b) { g_tally.div += 1; return Counting(a.v_ / b.v_); }

  friend bool operator<(Counting a, Counting b) { return a.v_ < b.v_; }
  friend bool operator>(Counting a, Counting b) { return a.v_ > b.v_; }
  friend bool operator<=(Counting a, Counting b) { return a.v_ <= b.v_; }
  friend bool operator>=(Counting a, Counting b) { return a.v_ >= b.v_; }
  friend bool operator==(Counting a, Counting b) { return a.v_ == b.v_; }
  friend bool operator!=(Counting a, Counting b) { return a.v_ != b.v_; }

  friend Counting sqrt(Counting a) { g_tally.sqrt_n += 1; return Counting(std::sqrt(a.v_)); }
  friend Counting fabs(Counting a) { return Counting(std::fabs(a.v_)); }
  friend Counting fmin(Counting a, Counting b) { return Counting(std::fmin(a.v_, b.v_)); }
  friend Counting fmax(Counting a, Counting b) { return Counting(std::fmax(a.v_, b.v_)); }
  friend Counting copysign(Counting a, Counting b) { return Counting(std::copysign(a.v_, b.v_)); }

 private:
  double v_ = 0.0;
};

inline double value_of(double v) { return v; }
inline double value_of(const Counting& v) { return v.value(); }

}  // namespace oracle

#endif
