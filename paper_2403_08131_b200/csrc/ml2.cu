// §8(f)1 ML-II: the Nelder-Mead state machine (host code; see ml2.cuh).  The batched driver
// (gp_fit_ml2) is in api.cu next to the fit it calls.
#include "ml2.cuh"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace gpbo {

uint64_t splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double ml2_uniform(uint64_t seed, int s, int k, int i, int dim, int starts) {
  const uint64_t c = 1ull + (uint64_t)i + (uint64_t)dim * ((uint64_t)k + (uint64_t)starts * s);
  return (double)(splitmix64(seed + 0x9E3779B97F4A7C15ull * c) >> 11) * 0x1.0p-53;
}

NelderMead::NelderMead(int dim, const double *x0, const double *lo, const double *hi, double step,
                       int iters)
    : dim_(dim), iters_(iters), x_((size_t)(dim + 1) * dim), f_(dim + 1), lo_(lo, lo + dim),
      hi_(hi, hi + dim), xbar_(dim), xr_(dim), xe_(dim), order_(dim + 1) {
  // initial simplex: x0 and x0 + step e_i (x0 - step e_i where that leaves the box)
  for (int v = 0; v <= dim; ++v) {
    double *x = &x_[(size_t)v * dim];
    for (int i = 0; i < dim; ++i) x[i] = x0[i];
    clamp_(x);
    if (v > 0) {
      const int i = v - 1;
      x[i] = x[i] + step <= hi_[i] ? x[i] + step : x[i] - step;
      clamp_(x);
    }
  }
  std::iota(order_.begin(), order_.end(), 0);
  req_ = x_;
  if (iters_ <= 0) phase_ = kInit;  // still evaluates the start simplex
}

void NelderMead::clamp_(double *x) const {
  for (int i = 0; i < dim_; ++i) x[i] = std::min(std::max(x[i], lo_[i]), hi_[i]);
}

void NelderMead::set_req_(const std::vector<double> &pts) { req_ = pts; }

// order_ = vertex indices by f ascending; stable on the previous order (a replaced vertex keeps
// the worst slot it took, so it sorts after any vertex with an equal f)
void NelderMead::sort_() {
  std::stable_sort(order_.begin(), order_.end(), [&](int a, int b) { return f_[a] < f_[b]; });
}

void NelderMead::next_iteration_() {
  if (++it_ >= iters_) {
    phase_ = kDone;
    req_.clear();
    return;
  }
  // reflect the worst vertex through the centroid of the others
  const int w = order_[dim_];
  for (int i = 0; i < dim_; ++i) {
    double c = 0.0;
    for (int v = 0; v < dim_; ++v) c += x_[(size_t)order_[v] * dim_ + i];
    xbar_[i] = c / dim_;
  }
  for (int i = 0; i < dim_; ++i) xr_[i] = 2.0 * xbar_[i] - x_[(size_t)w * dim_ + i];  // (1+rho) xbar - rho x_w
  clamp_(xr_.data());
  phase_ = kReflect;
  set_req_(xr_);
}

void NelderMead::deliver(const double *f) {
  const int w = order_[dim_];
  auto accept = [&](const std::vector<double> &x, double fx) {
    for (int i = 0; i < dim_; ++i) x_[(size_t)w * dim_ + i] = x[i];
    f_[w] = fx;
    sort_();
    next_iteration_();
  };
  auto shrink = [&]() {
    const int b = order_[0];
    std::vector<double> pts;
    for (int v = 1; v <= dim_; ++v) {
      const int q = order_[v];
      for (int i = 0; i < dim_; ++i) {
        double &xi = x_[(size_t)q * dim_ + i];
        xi = x_[(size_t)b * dim_ + i] + 0.5 * (xi - x_[(size_t)b * dim_ + i]);
        pts.push_back(xi);
      }
    }
    phase_ = kShrink;
    set_req_(pts);
  };
  switch (phase_) {
    case kInit: {
      for (int v = 0; v <= dim_; ++v) f_[v] = f[v];
      f0_ = f_[0];
      sort_();
      if (iters_ <= 0) { phase_ = kDone; req_.clear(); return; }
      it_ = -1;
      next_iteration_();
      return;
    }
    case kReflect: {
      fr_ = f[0];
      const double fb = f_[order_[0]], fsw = f_[order_[dim_ - 1]], fw = f_[w];
      if (fb <= fr_ && fr_ < fsw) { accept(xr_, fr_); return; }
      if (fr_ < fb) {  // expansion
        for (int i = 0; i < dim_; ++i) xe_[i] = 3.0 * xbar_[i] - 2.0 * x_[(size_t)w * dim_ + i];
        clamp_(xe_.data());
        phase_ = kExpand;
        set_req_(xe_);
        return;
      }
      if (fr_ < fw) {  // outside contraction
        for (int i = 0; i < dim_; ++i) xe_[i] = 1.5 * xbar_[i] - 0.5 * x_[(size_t)w * dim_ + i];
        clamp_(xe_.data());
        phase_ = kContractOut;
      } else {  // inside contraction
        for (int i = 0; i < dim_; ++i) xe_[i] = 0.5 * xbar_[i] + 0.5 * x_[(size_t)w * dim_ + i];
        phase_ = kContractIn;
      }
      set_req_(xe_);
      return;
    }
    case kExpand:
      if (f[0] < fr_) accept(xe_, f[0]); else accept(xr_, fr_);
      return;
    case kContractOut:
      if (f[0] <= fr_) accept(xe_, f[0]); else shrink();
      return;
    case kContractIn:
      if (f[0] < f_[w]) accept(xe_, f[0]); else shrink();
      return;
    case kShrink:
      for (int v = 1; v <= dim_; ++v) f_[order_[v]] = f[v - 1];
      sort_();
      next_iteration_();
      return;
    case kDone:
      return;
  }
}

}  // namespace gpbo
