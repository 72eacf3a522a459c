// Host side of §8(f)1 ML-II hyper-parameter fitting: multi-start Nelder-Mead in log space
// ("Nelder-Mead in log-space from 8 seeded starts, 200 iterations each; bounds
// lengthscale in [1e-3, 10], signal in [1e-3, 1e3], noise in [1e-6, 1]") maximising the log
// marginal likelihood that the fit kernel computes (fit.cu; the GP training the
// paper names as the O(N^3) cost).  Every objective evaluation is one search of a batched gp_fit
// launch: all (search, start) simplices advance together, one batched fit per round.
#pragma once
#include <cstdint>
#include <vector>

namespace gpbo {

// splitmix64 finaliser (Steele, Lea, Flood 2014): the start-point generator's mixing function.
uint64_t splitmix64(uint64_t z);
// Uniform [0, 1) double of coordinate i of start k of search s: 53 bits of
// splitmix64(seed + 0x9E3779B97F4A7C15 * (1 + i + dim * (k + starts * s))).
double ml2_uniform(uint64_t seed, int s, int k, int i, int dim, int starts);

// One Nelder-Mead simplex (minimises f = -LML) as a resumable state machine: request() returns
// the points (row-major, dim each) it needs evaluated next, deliver() takes their f values.
// Coefficients: reflection 1, expansion 2, contraction 1/2, shrink 1/2 (Nelder & Mead 1965;
// Lagarias et al. 1998 ordering: stable sort by f, a new vertex goes after its equals).  Points
// are clamped to the box [lo, hi].  Exactly `iters` iterations; no tolerance stop.
class NelderMead {
 public:
  NelderMead(int dim, const double *x0, const double *lo, const double *hi, double step, int iters);
  bool done() const { return phase_ == kDone; }
  const std::vector<double> &request() const { return req_; }
  void deliver(const double *f);
  // best vertex so far (after every delivery)
  const double *best_x() const { return &x_[(size_t)order_[0] * dim_]; }
  double best_f() const { return f_[order_[0]]; }
  double start_f() const { return f0_; }

 private:
  enum Phase { kInit, kReflect, kExpand, kContractOut, kContractIn, kShrink, kDone };
  void sort_();
  void next_iteration_();
  void clamp_(double *x) const;
  void set_req_(const std::vector<double> &pts);
  int dim_, iters_, it_ = 0;
  Phase phase_ = kInit;
  std::vector<double> x_, f_, lo_, hi_, xbar_, xr_, xe_, req_;
  std::vector<int> order_;
  double fr_ = 0.0, f0_ = 0.0;
};

}  // namespace gpbo
