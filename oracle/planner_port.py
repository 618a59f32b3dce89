"""ORACLE (test infrastructure only -- never imported by the product path).

Pure-Python restatement of the reference load-balancing planner, used as the
checker for the product planner (libmoeplan_b200.so) and for the GPU routing
kernels.  Each function cites the reference code it restates.  It is pinned
(tests/test_oracle_pinned.py) against (a) the golden vectors of the reference's
own unit tests (/root/reference/proj/tests/planner_test.cpp, cost_test.cpp,
sim_test.cpp) and (b) the reference library itself built into oracle/_ref.

Only the planner stage has reference code; see oracle/layer_oracle.py for the
layer numerics (parity unpinned -- no reference exists for them).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence

MASK64 = (1 << 64) - 1


# ----------------------------------------------------------------- rng.hpp:24-85
def mix_seed(seed: int, a: int, b: int = 0) -> int:
    """rng.hpp:25-32 (splitmix64 finalizer over a salted sum)."""
    z = (seed + 0x9E3779B97F4A7C15 * (a + 1) + 0x3C6EF372FE94F82B * (b + 1)) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


class MT19937_64:
    """std::mt19937_64 (C++ [rand.predef]), the engine of rng.hpp:84."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & MASK64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64


class Rng:
    """rng.hpp:37-85."""

    def __init__(self, seed: int):
        self.e = MT19937_64(seed)

    def next_u64(self) -> int:
        return self.e()

    def next_unit(self) -> float:
        return (self.e() >> 11) * 2.0 ** -53

    def next_below(self, n: int) -> int:
        return (self.e() * n) >> 64

    def next_normal(self) -> float:
        u1 = 1.0 - self.next_unit()
        u2 = self.next_unit()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * 3.141592653589793 * u2)

    def next_gamma(self, alpha: float) -> float:
        if alpha < 1.0:
            u = 1.0 - self.next_unit()
            return self.next_gamma(alpha + 1.0) * math.pow(u, 1.0 / alpha)
        d = alpha - 1.0 / 3.0
        c = 1.0 / math.sqrt(9.0 * d)
        while True:
            x = self.next_normal()
            t = 1.0 + c * x
            if t <= 0.0:
                continue
            v = t * t * t
            u = 1.0 - self.next_unit()
            x2 = x * x
            if u < 1.0 - 0.0331 * x2 * x2:
                return d * v
            if math.log(u) < 0.5 * x2 + d * (1.0 - v + math.log(v)):
                return d * v


class PlannerError(ValueError):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ------------------------------------------------------------- topology.hpp:26-75
@dataclass(frozen=True)
class Topology:
    n_nodes: int
    devices_per_node: int
    b_intra: float
    b_inter: float

    @property
    def n_devices(self) -> int:
        return self.n_nodes * self.devices_per_node

    def node_of(self, d: int) -> int:
        return d // self.devices_per_node

    def link_bandwidth(self, i: int, k: int) -> float:
        if i == k:
            return math.inf
        return self.b_intra if self.node_of(i) == self.node_of(k) else self.b_inter


@dataclass
class CostParams:
    v_comm: float
    v_comp: float
    b_comp: float
    f_ckpt: int = 0


def check_shape(n: int, e: int, c: int) -> None:
    """planner.cpp:29-43."""
    if n <= 0 or e <= 0 or c <= 0:
        raise PlannerError("invalid_argument", "planner: dimensions must be positive")
    if e > n * c:
        raise PlannerError("infeasible", f"planner: {e} experts exceed {n * c} device slots")
    if c > e:
        raise PlannerError("infeasible", f"planner: capacity {c} exceeds the expert count")


def _ratio_greater(a: float, b: int, c: float, d: int) -> bool:
    """planner.cpp:46-48 -- a/b > c/d evaluated as a*d > c*b in doubles."""
    return a * d > c * b


# ------------------------------------------------------------ planner.cpp:52-95
def replica_allocation(loads: Sequence[float], n: int, e: int, c: int) -> List[int]:
    check_shape(n, e, c)
    if len(loads) != e:
        raise PlannerError("invalid_argument", "replica_allocation: loads size disagrees with n_experts")
    for x in loads:
        if not (x >= 0.0):
            raise PlannerError("invalid_argument", "replica_allocation: loads must be non-negative")
    reps = [1] * e
    for _ in range(n * c - e):
        best = -1
        for j in range(e):
            if reps[j] >= n:
                continue
            if best < 0 or _ratio_greater(loads[j], reps[j], loads[best], reps[best]):
                best = j
        reps[best] += 1
    return reps


# ----------------------------------------------------------- planner.cpp:97-215
def expert_relocation(reps: Sequence[int], loads: Sequence[float], topo: Topology, c: int):
    """Returns the layout as a list of E rows of N 0/1 ints."""
    n = topo.n_devices
    e = len(reps)
    check_shape(n, e, c)
    order = []
    for j in range(e):
        order += [j] * reps[j]
    import functools

    def cmp(a, b):  # sort 120-129
        if _ratio_greater(loads[a], reps[a], loads[b], reps[b]):
            return -1
        if _ratio_greater(loads[b], reps[b], loads[a], reps[a]):
            return 1
        return (a > b) - (a < b)

    order.sort(key=functools.cmp_to_key(cmp))
    A = [[0] * n for _ in range(e)]
    used = [0] * n
    dload = [0.0] * n
    placed = [[] for _ in range(n)]
    ncount = [[0] * topo.n_nodes for _ in range(e)]

    def commit(j, share, d):
        A[j][d] = 1
        used[d] += 1
        dload[d] += share
        placed[d].append((j, share))
        ncount[j][topo.node_of(d)] += 1

    def select(j):  # 153-176
        counts = ncount[j]
        for level in sorted(set(counts)):
            best = -1
            for node in range(topo.n_nodes):
                if counts[node] != level:
                    continue
                for d in range(node * topo.devices_per_node, (node + 1) * topo.devices_per_node):
                    if used[d] < c and not A[j][d] and (best == -1 or dload[d] < dload[best]):
                        best = d
            if best != -1:
                return best
        return -1

    def repair(j):  # 181-201
        for d in range(n):
            if used[d] >= c:
                continue
            for donor in range(n):
                if donor == d or A[j][donor] or used[donor] < c:
                    continue
                for p, (mj, ml) in enumerate(placed[donor]):
                    if A[mj][d]:
                        continue
                    A[mj][donor] = 0
                    used[donor] -= 1
                    dload[donor] -= ml
                    ncount[mj][topo.node_of(donor)] -= 1
                    del placed[donor][p]
                    commit(mj, ml, d)
                    return donor
        return -1

    for j in order:
        d = select(j)
        if d == -1:
            d = repair(j)
        if d == -1:
            raise PlannerError("internal", f"expert_relocation: no placement for expert {j}")
        commit(j, loads[j] / reps[j], d)
    return A


# ---------------------------------------------------------- planner.cpp:217-236
def perturb_replicas(reps: Sequence[int], n: int, rng: Rng) -> List[int]:
    donors = [j for j, r in enumerate(reps) if r > 1]
    if not donors:
        return list(reps)
    donor = donors[rng.next_below(len(donors))]
    recips = [j for j, r in enumerate(reps) if j != donor and r < n]
    if not recips:
        return list(reps)
    rec = recips[rng.next_below(len(recips))]
    out = list(reps)
    out[donor] -= 1
    out[rec] += 1
    return out


# ---------------------------------------------------------- planner.cpp:238-287
def lite_routing(R, A, topo: Topology):
    """Returns sorted entries [(src, expert, dst, tokens)]."""
    n = len(R)
    e = len(R[0])
    hosts = [[d for d in range(n) if A[j][d]] for j in range(e)]
    entries = []
    for i in range(n):
        node = topo.node_of(i)
        for j in range(e):
            tokens = int(R[i][j])
            if tokens == 0:
                continue
            local = [d for d in hosts[j] if topo.node_of(d) == node]
            targets = local if local else hosts[j]
            if not targets:
                raise PlannerError("infeasible", f"lite_routing: expert {j} has load but no replica")
            share, extra = divmod(tokens, len(targets))
            for t, d in enumerate(targets):
                amt = share + (1 if t < extra else 0)
                if amt > 0:
                    entries.append((i, j, d, amt))
    return entries


# ---------------------------------------------------------------- cost.cpp:39-73
def time_cost(entries, n: int, topo: Topology, p: CostParams):
    recv = [0] * n
    secs = 0.0
    for (s, _j, d, tok) in entries:
        recv[d] += tok
        if s != d:
            secs += float(tok) / topo.link_bandwidth(s, d)
    t_comm = 4.0 * p.v_comm * secs
    fw = [p.v_comp * float(r) / p.b_comp for r in recv]
    t_comp = (3.0 + p.f_ckpt) * max(fw + [0.0])
    return {"t_comm": t_comm, "t_comp": t_comp, "t_total": t_comm + t_comp, "recv": recv}


# ---------------------------------------------------------- planner.cpp:289-307
def static_ep_layout(n: int, e: int, c: int):
    check_shape(n, e, c)
    A = [[0] * n for _ in range(e)]
    for s in range(n * c):
        A[s % e][s // c] = 1
    return A


def even_replicas(n: int, e: int, c: int) -> List[int]:
    reps = [(n * c) // e] * e
    for j in range((n * c) % e):
        reps[j] += 1
    return reps


def even_replication_layout(topo: Topology, e: int, c: int):
    check_shape(topo.n_devices, e, c)
    return expert_relocation(even_replicas(topo.n_devices, e, c), [1.0] * e, topo, c)


# ---------------------------------------------------------- planner.cpp:309-414
def aggregate_history(history, mode: str = "last", ema_decay: float = 0.5):
    if not history:
        raise PlannerError("invalid_argument", "aggregate_history: empty history")
    if mode == "last":
        return [[float(v) for v in row] for row in history[-1]]
    w = None
    for R in history:
        if w is None:
            w = [[float(v) for v in row] for row in R]
        else:
            w = [[ema_decay * float(R[i][j]) + (1.0 - ema_decay) * w[i][j] for j in range(len(R[0]))]
                 for i in range(len(R))]
    return w


def _llround(x: float) -> int:
    """std::llround: nearest integer, halves away from zero."""
    if x < 0:
        return -_llround(-x)
    f = math.floor(x)
    return int(f) + (1 if x - f >= 0.5 else 0)


@dataclass
class SearchSpec:
    epsilon: int = 2
    seed: int = 0
    history_mode: str = "last"
    ema_decay: float = 0.5


def plan_layout(history, topo: Topology, params: CostParams, c: int, spec: SearchSpec = None):
    spec = spec or SearchSpec()
    if spec.epsilon < 2:
        raise PlannerError("invalid_argument", "plan_layout: epsilon must be at least 2")
    W = aggregate_history(history, spec.history_mode, spec.ema_decay)
    n, e = len(W), len(W[0])
    check_shape(n, e, c)
    loads = [0.0] * e
    for i in range(n):
        for j in range(e):
            loads[j] += W[i][j]
    cands = [replica_allocation(loads, n, e, c), even_replicas(n, e, c)]
    rng = Rng(mix_seed(spec.seed, 0x706C616E))
    while len(cands) < spec.epsilon:
        base = cands[rng.next_below(len(cands))]
        cands.append(perturb_replicas(base, n, rng))
    score = [[_llround(v) for v in row] for row in W]
    best, best_cost = None, math.inf
    for reps in cands:
        A = expert_relocation(reps, loads, topo, c)
        cost = time_cost(lite_routing(score, A, topo), n, topo, params)["t_total"]
        if cost < best_cost:
            best, best_cost = A, cost
    return best


# --------------------------------------------------------------- sim.cpp:99-149
def lagged_layouts(records, topo: Topology, params: CostParams, c: int, spec: SearchSpec, layer: int,
                   scheduler: str = "laer"):
    """Layouts used at each step of one layer: step 0 = initial layout, step p
    = plan_layout(records[:p]) for laer (one-iteration lag)."""
    n = len(records[0])
    e = len(records[0][0])
    init = static_ep_layout(n, e, c) if scheduler == "static_ep" else even_replication_layout(topo, e, c)
    layer_spec = SearchSpec(spec.epsilon, mix_seed(spec.seed, 0x6C617972, layer), spec.history_mode, spec.ema_decay)
    out = []
    for p in range(len(records)):
        if p > 0 and scheduler == "laer":
            out.append(plan_layout(records[:p], topo, params, c, layer_spec))
        else:
            out.append(init)
    return out
