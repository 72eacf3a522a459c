"""Oracle of SURVEY.md §8(f)3, the interdependence planner -- TEST INFRASTRUCTURE ONLY (same rules
as oracle/gp.py; no code shared with the library's planner.cu).

Written from PAPER.md §IV.B-D (L185-260), §VIII (L455-567) and SPEC.md's planner module
(L228-325):

* influence(p -> r) = (1/V) sum_i |(t_base - t_i) / t_base|   (§IV.B), over the valid
  variations only; NaN when none is valid ("unknown").
* Global stage (§VIII): routines that are outer regions (have child routines) or have
  no metric of their own get stage-1 searches (against their metric / the total objective); a
  child-owned parameter at or above the cut-off on its parent and on >= 2 sibling children is
  pulled up into the parent's search.
* Shared kernels (§IV step 5, L545): a parameter owned by several routines is owned by the one
  where its influence is highest (ties: the lower routine index).
* Partition (§IV.C): a cross edge (owner q -> routine r, both children) at or above the
  cut-off merges q and r when the parameter must keep one value, else the parameter is also
  tuned in r's search ("tune affected parameters twice").  Merged groups = connected components.
* Dimension cap (§IV step 4, L167; §IV.D): above dim_cap parameters, keep the dim_cap with
  the highest influence (max over the search's routines; ties: lower parameter index).
* Budget (§IV.D): max(floor, multiplier x dims).
"""
from __future__ import annotations

import math


def influence(baseline, variations, valid=None):
    """baseline[r]; variations[p][i][r]; valid[p][i] or None -> matrix[r][p] (lists)."""
    R = len(baseline)
    P = len(variations)
    M = [[math.nan] * P for _ in range(R)]
    for r in range(R):
        for p in range(P):
            acc, cnt = 0.0, 0
            for i in range(len(variations[p])):  # plain left-to-right sum (not math.fsum)
                if valid is None or valid[p][i]:
                    acc += abs((baseline[r] - variations[p][i][r]) / baseline[r])
                    cnt += 1
            if cnt:
                M[r][p] = acc / cnt
    return M


def plan(matrix, owners, parent=None, has_metric=None, shared=None, cutoff=0.25, dim_cap=10,
         budget_mult=10, budget_floor=10):
    R = len(matrix)
    P = len(matrix[0])
    parent = parent or [-1] * R
    has_metric = has_metric or [1] * R
    shared = shared or [1] * P

    def w(r, p):
        v = matrix[r][p]
        return 0.0 if v is None or not math.isfinite(v) else v

    children = {r: [c for c in range(R) if parent[c] == r] for r in range(R)}
    child = [bool(has_metric[r]) and not children[r] for r in range(R)]
    own = []
    for p in range(P):
        cands = sorted(owners[p])
        own.append(max(cands, key=lambda r: (w(r, p), -r)))
    for p in range(P):
        q = own[p]
        if not child[q] or parent[q] < 0:
            continue
        par = parent[q]
        sibs = [c for c in children[par] if child[c] and w(c, p) >= cutoff]
        if w(par, p) >= cutoff and len(sibs) >= 2:
            own[p] = par
    # graph over child routines: merge edges and duplicates
    adj = {r: set() for r in range(R) if child[r]}
    extra = {r: [] for r in range(R)}
    for r in range(R):
        if not child[r]:
            continue
        for p in range(P):
            q = own[p]
            if q == r or not child[q] or not (w(r, p) >= cutoff):
                continue
            if shared[p]:
                adj[q].add(r)
                adj[r].add(q)
            else:
                extra[r].append(p)
    comp = {}
    for r in sorted(adj):
        if r in comp:
            continue
        stack, members = [r], []
        comp[r] = r
        while stack:
            x = stack.pop()
            members.append(x)
            for y in adj[x]:
                if y not in comp:
                    comp[y] = r
                    stack.append(y)
    searches = []
    for r in range(R):  # stage 1: global routines owning parameters
        if child[r]:
            continue
        ps = [p for p in range(P) if own[p] == r]
        if ps:
            searches.append(dict(stage=1, target=r if has_metric[r] else -1, routines=[r],
                                 params=ps))
    for root in sorted(set(comp.values())):  # stage 2: components, by lowest routine
        mem = sorted(x for x in comp if comp[x] == root)
        ps = sorted(set(p for p in range(P) if own[p] in mem) |
                    set(p for x in mem for p in extra[x]))
        if ps:
            searches.append(dict(stage=2, target=root, routines=mem, params=ps))
    for s in searches:
        if len(s["params"]) > dim_cap:
            infl = {p: max(w(r, p) for r in s["routines"]) for p in s["params"]}
            keep = sorted(s["params"], key=lambda p: (-infl[p], p))[:dim_cap]
            s["params"] = sorted(keep)
        s["budget"] = max(budget_floor, budget_mult * len(s["params"]))
    tuned = set(p for s in searches for p in s["params"])
    dropped = [p for p in range(P) if p not in tuned]
    return [dict(stage=s["stage"], target=s["target"], budget=s["budget"], params=s["params"])
            for s in searches], dropped
