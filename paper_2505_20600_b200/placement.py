"""Mask-aware request placement across GPU replicas (§8(e)).

Host-side policy of the multi-GPU partition: requests are independent (attention and the K/V
merge are per request), so the box runs one full replica per GPU and a dispatcher
assigns each arriving request to one replica.  This module follows the paper:

* linear latency models fitted offline: FLOPs -> compute latency, bytes -> cache-load latency
  ("linear regression models ... R^2 of 0.99");            LatencyModel, fit_ols
* per-request work from the Table 1 cost model:   step_flops,
  step_load_bytes (K/V variant, compacted transfer)
* the block-level pipeline recurrence of Algorithm 1 as the batch latency
  estimate ("dp(new_batch, Comp, Load)" in Algorithm 2);                   algorithm1
* Algorithm 2: candidates = workers with slack in their running batch; cost =
  pipeline latency of worker.running_batch + req; assign to the argmin (ties -> lowest id,
  S:490); if no worker has slack, all workers are candidates.    Placement.route

Nothing here touches a GPU; the dispatcher sends request descriptors to worker processes over
a torch.distributed (gloo) group (dispatch_gloo), the in-box stand-in for the paper's ZeroMQ
(P:793-794).  There is no collective on the step path.
"""
from __future__ import annotations

import dataclasses
import itertools
from typing import Dict, List, Optional, Sequence, Tuple


# ---------------------------------------------------------------------------------------
# Linear latency models
# ---------------------------------------------------------------------------------------
def fit_ols(xs: Sequence[float], ys: Sequence[float]) -> Tuple[float, float, float]:
    """Ordinary least squares y = slope x + intercept; returns (slope, intercept, r2).
    Raises ValueError when the x values are all equal (S:195-197 'degenerate')."""
    n = len(xs)
    if n < 2 or len(ys) != n:
        raise ValueError("fit needs >= 2 points")
    mx = sum(xs) / n
    my = sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    if sxx == 0.0:
        raise ValueError("fit-error: degenerate x (all equal)")
    sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    slope = sxy / sxx
    icpt = my - slope * mx
    ss_tot = sum((y - my) ** 2 for y in ys)
    ss_res = sum((y - (slope * x + icpt)) ** 2 for x, y in zip(xs, ys))
    r2 = 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0
    return slope, icpt, r2


@dataclasses.dataclass
class LatencyModel:
    comp_slope: float      # seconds per FLOP
    comp_intercept: float  # seconds
    load_slope: float      # seconds per byte
    load_intercept: float  # seconds
    r2_comp: float = 1.0
    r2_load: float = 1.0

    def comp(self, flops: float) -> float:
        return self.comp_slope * flops + self.comp_intercept if flops > 0 else 0.0

    def load(self, nbytes: float) -> float:
        return self.load_slope * nbytes + self.load_intercept if nbytes > 0 else 0.0

    @classmethod
    def fitted(cls, comp_pts, load_pts) -> "LatencyModel":
        a, b, r = fit_ols([p[0] for p in comp_pts], [p[1] for p in comp_pts])
        c, d, s = fit_ols([p[0] for p in load_pts], [p[1] for p in load_pts])
        return cls(a, b, c, d, r, s)


# ---------------------------------------------------------------------------------------
# Table 1 work per request-step (per block), K/V variant
# ---------------------------------------------------------------------------------------
def block_flops(desc, n_m: int) -> float:
    """Algorithmic FLOPs of one block for one request with n_m masked tokens: every
    projection / FF scales with the query rows (L_txt + n_m), attention with rows x L
    (Table 1 rows XW, (XW1)W2, QK^T)."""
    H, F, L = desc.hidden, desc.mlp_hidden, desc.txt_len + desc.grid_h * desc.grid_w
    rows = desc.txt_len + n_m
    lin = 2 * rows * (3 * H * H + H * H + 2 * H * F)  # double and single blocks are equal per row
    att = 4 * rows * L * H
    return float(lin + att)


def block_load_bytes(desc, n_m: int, elem_bytes: int = 2) -> float:
    """Cached K and V of the unmasked tokens of one block (cache shape (1-m)L x H per tensor,
    Table 1; 'doubles' the Y cache)."""
    L_img = desc.grid_h * desc.grid_w
    return float(2 * (L_img - n_m) * desc.hidden * elem_bytes) if 0 < n_m < L_img else 0.0


# ---------------------------------------------------------------------------------------
# Algorithm 1: bubble-free pipeline recurrence
# ---------------------------------------------------------------------------------------
def algorithm1(N: int, c_w: float, c_wo: float, l: float, tie: str = "<="):
    """Greedy recurrence of Algorithm 1, verbatim: for block i, caching finishes at
    max(load_{i-1} + L, comp_{i-1}) + C_w; computing densely at comp_{i-1} + C_w/o.  'tie'
    selects the paper's '<=' (cache on ties) or the strict '<' variant.
    Returns (use_cache[N], comp[N+1], load[N+1], pipeline_latency)."""
    comp = [0.0] * (N + 1)
    load = [0.0] * (N + 1)
    use = [False] * N
    for i in range(1, N + 1):
        cached = max(load[i - 1] + l, comp[i - 1]) + c_w
        dense = comp[i - 1] + c_wo
        take = cached <= dense if tie == "<=" else cached < dense
        if take:
            load[i] = load[i - 1] + l
            comp[i] = cached
            use[i - 1] = True
        else:
            load[i] = load[i - 1]
            comp[i] = dense
            use[i - 1] = False
    return use, comp, load, comp[N]


def pipeline_latency(plan: Sequence[bool], c_w: float, c_wo: float, l: float) -> float:
    """Latency of a given plan under the same two-lane model (used by the exact planner)."""
    comp = load = 0.0
    for u in plan:
        if u:
            load = load + l
            comp = max(load, comp) + c_w
        else:
            comp = comp + c_wo
    return comp


def exact_plan(N: int, c_w: float, c_wo: float, l: float):
    """Brute force over all 2^N plans (the planner's test oracle)."""
    best = None
    for plan in itertools.product([False, True], repeat=N):
        t = pipeline_latency(plan, c_w, c_wo, l)
        if best is None or t < best[1] - 1e-12:
            best = (list(plan), t)
    return best


# ---------------------------------------------------------------------------------------
# Algorithm 2: mask-aware routing
# ---------------------------------------------------------------------------------------
@dataclasses.dataclass
class Worker:
    wid: int
    running: List[int] = dataclasses.field(default_factory=list)  # n_m of each member


class Placement:
    """Algorithm 2 over n_workers GPU replicas.  uplinks (optional): the host-link uplink each
    worker's GPU sits behind (e.g. GPUs sharing a PCIe switch, from `nvidia-smi topo -m` and the
    concurrent-H2D probe, tools/probe_box.py --concurrent), with uplink_load_slope the seconds
    per byte of one uplink shared by all its GPUs (SURVEY §8(e) "add a per-uplink term to a_l so
    the policy pairs high-m with low-m requests on siblings").  A worker's per-block load time is
    then max(Load(own bytes), uplink_load_slope * bytes of every worker on its uplink)."""

    def __init__(self, desc, model: LatencyModel, n_workers: int, max_batch: int = 8,
                 elem_bytes: int = 2, tie: str = "<=", uplinks: Optional[Sequence[int]] = None,
                 uplink_load_slope: float = 0.0):
        self.desc, self.model, self.max_batch = desc, model, max_batch
        self.elem_bytes, self.tie = elem_bytes, tie
        self.workers = [Worker(i) for i in range(n_workers)]
        self.N = desc.n_double + desc.n_single
        self.L_img = desc.grid_h * desc.grid_w
        self.uplinks = list(uplinks) if uplinks is not None else None
        self.uplink_load_slope = uplink_load_slope

    def _bytes(self, batch: Sequence[int]) -> float:
        return sum(block_load_bytes(self.desc, n, self.elem_bytes) for n in batch)

    def batch_latency(self, batch: Sequence[int], wid: Optional[int] = None) -> float:
        """dp(batch, Comp, Load): Algorithm 1 over the blocks of one step of the batch, with
        C_w = Comp(sum of masked-batch FLOPs), C_w/o = Comp(dense FLOPs of the batch) and
        L = Load(sum of cached bytes) per block (the batch sums compute and bytes); with
        uplinks, L is at least the shared uplink's time for all its workers' bytes."""
        if not batch:
            return 0.0
        f_w = sum(block_flops(self.desc, n) for n in batch)
        f_wo = sum(block_flops(self.desc, self.L_img) for _ in batch)
        b = self._bytes(batch)
        load = self.model.load(b)
        if self.uplinks is not None and wid is not None and self.uplink_load_slope > 0 and b > 0:
            shared = b + sum(self._bytes(w.running) for w in self.workers
                             if w.wid != wid and self.uplinks[w.wid] == self.uplinks[wid])
            load = max(load, self.uplink_load_slope * shared)
        return algorithm1(self.N, self.model.comp(f_w), self.model.comp(f_wo), load, self.tie)[3]

    def calc_cost(self, n_m: int, w: Worker) -> float:
        """Algorithm 2's cost: the step latency of w's batch with the request added; with
        uplinks, the slowest step among the workers behind w's uplink (adding bytes to w also
        slows its siblings' loads)."""
        if self.uplinks is None or self.uplink_load_slope <= 0:
            return self.batch_latency(w.running + [n_m], w.wid)
        w.running.append(n_m)
        try:
            return max(self.batch_latency(o.running, o.wid) for o in self.workers
                       if self.uplinks[o.wid] == self.uplinks[w.wid])
        finally:
            w.running.pop()

    def route(self, n_m: int) -> int:
        cands = [w for w in self.workers if len(w.running) < self.max_batch] or self.workers
        best = min(cands, key=lambda w: (self.calc_cost(n_m, w), w.wid))
        best.running.append(n_m)
        return best.wid

    def finish(self, wid: int, n_m: int):
        self.workers[wid].running.remove(n_m)


# ---------------------------------------------------------------------------------------
# Multi-process dispatch over a gloo process group (control plane only)
# ---------------------------------------------------------------------------------------
def dispatch_gloo(requests: Optional[List[Tuple[int, int]]], placement: Optional[Placement]) -> List[Tuple[int, int]]:
    """Rank 0 routes every (request id, n_m) with Algorithm 2 and sends each worker its
    descriptors; returns this rank's list.  Collective on the CPU control plane only."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [None]
    if rank == 0:
        per = [[] for _ in range(world)]
        for rid, n_m in requests:
            per[placement.route(n_m)].append((rid, n_m))
        obj = [per]
    dist.broadcast_object_list(obj, src=0)
    return obj[0][rank]
