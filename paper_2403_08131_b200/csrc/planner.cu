// the interdependence planner that emits the batch of sub-searches the GPU
// path fits and scores (host code; cheap).  PAPER.md §IV.B-D (L185-260) and §VIII (L455-567):
//
//  * influence (§IV.B): variability of routine r under the V individual variations of
//    parameter p = (1/V) sum_i |(t_base - t_i) / t_base| -- one row per measured routine
//    (invalid variations are skipped and the divisor reduced);
//  * interdependence graph (§IV.C): routines are vertices, parameter -> routine edges carry
//    the variability, edges below the cut-off are pruned (25 % synthetic L254, 10 % RT-TDDFT
//    L543);
//  * global stage (§VIII): parameters of a routine without a metric of its own (the MPI
//    grid: against the total objective) and of an outer region (Slater determinant: nbatches,
//    nstreams) form stage-1 searches, their results fixed for stage 2; a child-owned parameter
//    above the cut-off on the parent and on >= 2 children is pulled up into the parent's search;
//  * shared kernels (§IV step 5, L545): a parameter owned by several routines (one kernel used in
//    several regions, one value) is tuned only where its variability is highest;
//  * merge / tune twice (§IV.C): a surviving cross edge whose parameter must keep one value
//    merges the two routines' searches (union-find; connected components); any other surviving
//    cross edge duplicates the parameter into the target routine's search;
//  * dimension cap (§IV step 4, L167, L249): a search with more than dim_cap parameters keeps the
//    dim_cap most influential (max over its routines) and fixes the rest at their defaults;
//  * budget (§IV.D): max(floor, multiplier x dims) evaluations.
// Ties resolve to the lower routine / parameter index everywhere (deterministic).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "../../include/gpbo.h"

namespace {

int uf_find(std::vector<int> &p, int x) {
  while (p[x] != x) x = p[x] = p[p[x]];
  return x;
}

void uf_union(std::vector<int> &p, int a, int b) {
  a = uf_find(p, a);
  b = uf_find(p, b);
  if (a == b) return;
  if (a < b) p[b] = a; else p[a] = b;  // the lower index is the root
}

}  // namespace

extern "C" {

gpbo_status gpbo_influence(int32_t R, int32_t P, int32_t V, const double *baseline,
                           const double *variations, const uint8_t *valid, double *matrix) {
  if (R < 1 || P < 1 || V < 1 || !baseline || !variations || !matrix) return GPBO_EINVAL;
  for (int r = 0; r < R; ++r)
    if (!(baseline[r] != 0.0) || !std::isfinite(baseline[r])) return GPBO_EINVAL;
  for (int r = 0; r < R; ++r)
    for (int p = 0; p < P; ++p) {
      double acc = 0.0;
      int ok = 0;
      for (int i = 0; i < V; ++i) {
        if (valid && !valid[(size_t)p * V + i]) continue;
        const double t = variations[((size_t)p * V + i) * R + r];
        acc += std::fabs((baseline[r] - t) / baseline[r]);
        ++ok;
      }
      matrix[(size_t)r * P + p] = ok ? acc / ok : NAN;  // all invalid: unknown, not 0
    }
  return GPBO_OK;
}

gpbo_status gpbo_plan(const gpbo_plan_args *a, gpbo_plan_out *o) {
  if (!a || !o || a->R < 1 || a->P < 1 || !a->parent || !a->has_metric || !a->owner_off ||
      !a->owners || !a->shared || !a->matrix || !o->search_stage || !o->search_target ||
      !o->search_budget || !o->search_dims || !o->tuned || !o->dropped || a->dim_cap < 1 ||
      !(a->cutoff >= 0.0))
    return GPBO_EINVAL;
  const int R = a->R, P = a->P;
  const double cut = a->cutoff;
  auto W = [&](int r, int p) {  // influence of p on r (unknown -> 0: no edge)
    const double v = a->matrix[(size_t)r * P + p];
    return std::isfinite(v) ? v : 0.0;
  };
  std::vector<int> nchild(R, 0);
  for (int r = 0; r < R; ++r) {
    if (a->parent[r] < -1 || a->parent[r] >= R) return GPBO_EINVAL;
    if (a->parent[r] >= 0) nchild[a->parent[r]]++;
  }
  for (int p = 0; p < P; ++p) {
    if (a->owner_off[p + 1] <= a->owner_off[p]) return GPBO_EINVAL;  // >= 1 owner
    for (int k = a->owner_off[p]; k < a->owner_off[p + 1]; ++k)
      if (a->owners[k] < 0 || a->owners[k] >= R) return GPBO_EINVAL;
  }
  // a routine is a "child" (a stage-2 search candidate) when it has a metric and no children;
  // the others are global: outer regions (stage-1 search against their metric) and routines
  // without a metric (stage-1 search against the total objective, target -1)
  auto is_child = [&](int r) { return a->has_metric[r] && nchild[r] == 0; };
  // ---- owner of every parameter (shared kernels: the owner where p's influence is highest)
  std::vector<int> owner(P);
  for (int p = 0; p < P; ++p) {
    int best = a->owners[a->owner_off[p]];
    for (int k = a->owner_off[p] + 1; k < a->owner_off[p + 1]; ++k) {
      const int r = a->owners[k];
      if (W(r, p) > W(best, p) || (W(r, p) == W(best, p) && r < best)) best = r;
    }
    owner[p] = best;
  }
  // ---- global stage: pull child-owned parameters up into the parent region's search
  for (int p = 0; p < P; ++p) {
    const int r0 = owner[p];
    if (!is_child(r0)) continue;
    const int par = a->parent[r0];
    if (par < 0 || W(par, p) < cut) continue;
    int above = 0;
    for (int r = 0; r < R; ++r)
      if (is_child(r) && a->parent[r] == par && W(r, p) >= cut) ++above;
    if (above >= 2) owner[p] = par;
  }
  // ---- partition of the child routines: merge along surviving one-value cross edges
  std::vector<int> uf(R);
  std::iota(uf.begin(), uf.end(), 0);
  std::vector<std::vector<int>> dup(R);  // tuned twice: parameter p also in routine r's search
  for (int r = 0; r < R; ++r) {
    if (!is_child(r)) continue;
    for (int p = 0; p < P; ++p) {
      const int q = owner[p];
      if (q == r || !is_child(q) || W(r, p) < cut) continue;
      if (a->shared[p]) uf_union(uf, q, r);
      else dup[r].push_back(p);
    }
  }
  // ---- searches: stage 1 (global routines in index order), then stage 2 (child components,
  // ordered by their lowest routine)
  const int maxs = R;  // at most one search per routine
  int ns = 0;
  std::fill(o->tuned, o->tuned + (size_t)maxs * P, (uint8_t)0);
  std::vector<int> search_of(R, -1);
  for (int stage = 1; stage <= 2; ++stage)
    for (int r = 0; r < R; ++r) {
      if (stage == 1 ? is_child(r) : (!is_child(r) || uf_find(uf, r) != r)) continue;
      bool any = false;
      for (int p = 0; p < P && !any; ++p)
        any = stage == 1 ? owner[p] == r : (is_child(owner[p]) && uf_find(uf, owner[p]) == r);
      if (!any && stage == 2) {  // a component may own only duplicated parameters
        for (int q = 0; q < R && !any; ++q)
          any = is_child(q) && uf_find(uf, q) == r && !dup[q].empty();
      }
      if (!any) continue;
      search_of[r] = ns;
      o->search_stage[ns] = stage;
      o->search_target[ns] = a->has_metric[r] ? r : -1;
      ++ns;
    }
  for (int r = 0; r < R; ++r)
    if (is_child(r) && search_of[r] < 0) search_of[r] = search_of[uf_find(uf, r)];
  for (int p = 0; p < P; ++p) {
    const int q = owner[p];
    const int s = search_of[is_child(q) ? uf_find(uf, q) : q];
    if (s >= 0) o->tuned[(size_t)s * P + p] = 1;
  }
  for (int r = 0; r < R; ++r)
    for (int p : dup[r]) {
      const int s = search_of[uf_find(uf, r)];
      if (s >= 0) o->tuned[(size_t)s * P + p] = 1;
    }
  // ---- dimension cap: keep the dim_cap most influential parameters of each search (max over
  // the search's routines; ties -> lower parameter index), the rest fixed at their defaults
  for (int s = 0; s < ns; ++s) {
    std::vector<int> mem;
    for (int r = 0; r < R; ++r) {
      const int root = is_child(r) ? uf_find(uf, r) : r;
      if (search_of[root] == s && (is_child(r) || root == r)) mem.push_back(r);
    }
    std::vector<int> ps;
    for (int p = 0; p < P; ++p)
      if (o->tuned[(size_t)s * P + p]) ps.push_back(p);
    if ((int)ps.size() > a->dim_cap) {
      std::vector<double> inf(P, 0.0);
      for (int p : ps)
        for (int r : mem) inf[p] = std::max(inf[p], W(r, p));
      std::stable_sort(ps.begin(), ps.end(), [&](int x, int y) { return inf[x] > inf[y]; });
      for (size_t i = a->dim_cap; i < ps.size(); ++i) o->tuned[(size_t)s * P + ps[i]] = 0;
      ps.resize(a->dim_cap);
    }
    o->search_dims[s] = (int32_t)ps.size();
    o->search_budget[s] = std::max(a->budget_floor, a->budget_mult * (int32_t)ps.size());
  }
  // every parameter is accounted for: tuned somewhere, or dropped (fixed at its default)
  for (int p = 0; p < P; ++p) {
    bool t = false;
    for (int s = 0; s < ns && !t; ++s) t = o->tuned[(size_t)s * P + p] != 0;
    o->dropped[p] = t ? 0 : 1;
  }
  o->nsearch = ns;
  return GPBO_OK;
}

}  // extern "C"
