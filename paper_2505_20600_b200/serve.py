"""Serving loop and policies: step-level continuous batching under Poisson
arrivals, routed across GPU workers by the mask-aware policy of Algorithm 2.

Paper passages this follows
* Step-level continuous batching: "once a request completes all steps of computation, it is
  immediately removed from the running batch; new requests can join the batch in just one
  step".  Static batching keeps "a fixed running batch size until the running
  batch completes".                                     Engine(policy=...)
* Pre/post-processing are disaggregated from the denoising lane: the engine's
  step loop only runs ig_edit_step; admission work (mask index build, latent upload) happens
  at step boundaries off the compute stream.
* Mask-aware routing (Algorithm 2) with linear latency models and the
  request-count / token-count balancing baselines it is compared with.
                                                       route_trace, simulate_cluster
* Metrics: mean and P95 request latency (nearest rank) and queueing time.  percentile

Host logic only (no arithmetic of the method): the per-step latency estimate reuses the
Algorithm-1 pipeline recurrence of placement.py; the GPU work is ig_edit_step.
"""
from __future__ import annotations

import dataclasses
import heapq
import math
from typing import Dict, List, Optional, Sequence

import numpy as np

from .placement import LatencyModel, algorithm1, block_flops, block_load_bytes


# ---------------------------------------------------------------------------------------
# metrics
# ---------------------------------------------------------------------------------------
def percentile(samples: Sequence[float], p: float) -> float:
    """Nearest-rank percentile: the ceil(p n)-th order statistic."""
    if len(samples) == 0:
        raise ValueError("invalid-argument: empty sample list")
    if not (0.0 < p <= 1.0):
        raise ValueError("invalid-argument: p must be in (0, 1]")
    s = sorted(samples)
    return s[max(1, math.ceil(p * len(s))) - 1]


def summarize(lat: Sequence[float], queue: Sequence[float]) -> Dict[str, float]:
    return {"n": len(lat), "mean_latency_s": float(np.mean(lat)) if lat else None,
            "p95_latency_s": percentile(lat, 0.95) if lat else None,
            "mean_queue_s": float(np.mean(queue)) if queue else None,
            "p95_queue_s": percentile(queue, 0.95) if queue else None}


# ---------------------------------------------------------------------------------------
# workload: Poisson arrivals with per-request mask ratios (S: workload module)
# ---------------------------------------------------------------------------------------
@dataclasses.dataclass
class Arrival:
    rid: int
    t: float      # arrival time (s) from the start of the run
    n_m: int      # masked image tokens


def poisson_trace(rate: float, n: int, L_img: int, seed: int = 0, lo: float = 0.05, hi: float = 0.60,
                  skew: Optional[str] = None) -> List[Arrival]:
    """n arrivals with exponential inter-arrival times of mean 1/rate; m ~ U[lo, hi] (the
    headline mix) or one of the skewed presets of SURVEY §8(d) config 4."""
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.exponential(1.0 / rate, n))
    if skew == "public":
        m = 0.05 + 0.55 * rng.beta(1.5, 4.5, n)
    elif skew == "own":
        m = 0.05 + 0.55 * rng.beta(1.0, 8.0, n)
    else:
        m = rng.uniform(lo, hi, n)
    return [Arrival(i, float(t[i]), max(1, int(round(m[i] * L_img)))) for i in range(n)]


# ---------------------------------------------------------------------------------------
# per-step latency estimate and Algorithm 2 cost
# ---------------------------------------------------------------------------------------
class StepModel:
    """Predicted latency of one denoising step of a batch: Algorithm 1's pipeline latency
    over the blocks with C_w = Comp(sum of masked FLOPs), C_w/o = Comp(dense FLOPs),
    L = Load(sum of cached bytes)."""

    def __init__(self, desc, model: LatencyModel, elem_bytes: int = 2, y_frac: float = 0.0):
        """y_frac: fraction of Y blocks of a hybrid cache (DESIGN reading 30): they move one
        plane instead of two and recompute the unmasked rows' K/V (4 n_u H^2 flops)."""
        self.desc, self.model, self.eb, self.y_frac = desc, model, elem_bytes, y_frac
        self.N = desc.n_double + desc.n_single
        self.L_img = desc.grid_h * desc.grid_w
        self._memo: Dict[tuple, float] = {}

    def step(self, batch: Sequence[int]) -> float:
        if not batch:
            return 0.0
        key = tuple(sorted(batch))
        v = self._memo.get(key)
        if v is None:
            H = self.desc.hidden
            f_w = sum(block_flops(self.desc, n) + self.y_frac * 4.0 * (self.L_img - n) * H * H for n in batch)
            f_wo = len(batch) * block_flops(self.desc, self.L_img)
            b = (1.0 - 0.5 * self.y_frac) * sum(block_load_bytes(self.desc, n, self.eb) for n in batch)
            v = algorithm1(self.N, self.model.comp(f_w), self.model.comp(f_wo), self.model.load(b))[3]
            self._memo[key] = v
        return v

    def drain_cost(self, members: Sequence[tuple]) -> float:
        """Cost of a batch as the sum over future step boundaries of the predicted step
        latency of the evolving batch, members leaving at their completion (SPEC scheduler
        design decision; Algorithm 2's CalcCost over a multi-step horizon).
        members: (n_m, remaining_steps)."""
        rem = sorted(members, key=lambda x: x[1])
        cost, done, live = 0.0, 0, [m for m in rem]
        while live:
            k = live[0][1] - done  # steps until the next member leaves
            cost += k * self.step([m[0] for m in live])
            done = live[0][1]
            live = [m for m in live if m[1] > done]
        return cost


@dataclasses.dataclass
class WorkerState:
    wid: int
    running: List[list] = dataclasses.field(default_factory=list)  # [n_m, remaining_steps, rid]
    queue: List[Arrival] = dataclasses.field(default_factory=list)
    t: float = 0.0           # time of the next step boundary
    assigned_tokens: int = 0


POLICIES = ("mask_aware", "request_count", "token_count")


def _route(ws: List[WorkerState], a: Arrival, policy: str, sm: StepModel, max_batch: int, n_steps: int) -> int:
    if policy == "request_count":
        return min(ws, key=lambda w: (len(w.running) + len(w.queue), w.wid)).wid
    if policy == "token_count":
        return min(ws, key=lambda w: (w.assigned_tokens, w.wid)).wid
    # Algorithm 2: candidates = workers with slack in the running batch (else all); cost =
    # predicted serving latency of running batch + queue + the new request
    cands = [w for w in ws if len(w.running) + len(w.queue) < max_batch] or ws

    def cost(w):
        mem = [(r[0], r[1]) for r in w.running] + [(q.n_m, n_steps) for q in w.queue] + [(a.n_m, n_steps)]
        return sm.drain_cost(mem)
    return min(cands, key=lambda w: (cost(w), w.wid)).wid


def simulate_cluster(trace: Sequence[Arrival], n_workers: int, policy: str, sm: StepModel,
                     max_batch: int = 8, n_steps: int = 28, batching: str = "continuous"):
    """Virtual-clock discrete-event simulation of the cluster under the latency model: each
    arrival is routed on arrival (Algorithm 2 or a baseline), workers run step-level
    continuous (or static) batching.  Returns (assignment {rid: wid}, per-request records
    {rid: (arrive, admit, done)})."""
    if policy not in POLICIES:
        raise ValueError(f"unknown policy {policy}")
    ws = [WorkerState(i) for i in range(n_workers)]
    assign: Dict[int, int] = {}
    rec: Dict[int, list] = {}
    pending = sorted(trace, key=lambda a: (a.t, a.rid))
    i = 0
    # advance all workers' step loops up to time T (processing step boundaries in order)
    def advance(T):
        heap = [(w.t, w.wid) for w in ws if w.running or w.queue]
        heapq.heapify(heap)
        while heap:
            t, wid = heapq.heappop(heap)
            w = ws[wid]
            if t > T:
                break
            # step boundary at time t: admit
            if batching == "continuous" or not w.running:
                while w.queue and len(w.running) < max_batch and w.queue[0].t <= t:
                    q = w.queue.pop(0)
                    w.running.append([q.n_m, n_steps, q.rid])
                    rec[q.rid][1] = t
            if not w.running:
                w.t = w.queue[0].t if w.queue else t
                if w.queue:
                    heapq.heappush(heap, (w.t, wid))
                continue
            dt = sm.step([r[0] for r in w.running])
            w.t = t + dt
            for r in w.running:
                r[1] -= 1
            for r in [r for r in w.running if r[1] == 0]:
                rec[r[2]][2] = w.t
                w.running.remove(r)
            heapq.heappush(heap, (w.t, wid))

    while i < len(pending):
        a = pending[i]
        advance(a.t)
        wid = _route(ws, a, policy, sm, max_batch, n_steps)
        w = ws[wid]
        assign[a.rid] = wid
        rec[a.rid] = [a.t, None, None]
        w.queue.append(a)
        w.assigned_tokens += a.n_m
        if not w.running and len(w.queue) == 1:
            w.t = max(w.t, a.t)
        i += 1
    advance(float("inf"))
    return assign, rec


def route_trace(trace: Sequence[Arrival], n_workers: int, sm: StepModel, policy: str = "mask_aware",
                max_batch: int = 8, n_steps: int = 28) -> Dict[int, int]:
    """The dispatcher's decisions for a whole trace (online, in arrival order; worker state
    tracked with the latency model between decisions)."""
    return simulate_cluster(trace, n_workers, policy, sm, max_batch, n_steps)[0]


def dispatch_trace(trace: Sequence[Arrival], sm: StepModel, policy: str = "mask_aware",
                   max_batch: int = 8, n_steps: int = 28) -> List[Arrival]:
    """Rank 0 routes every arrival (Algorithm 2 or a baseline) and broadcasts the decisions
    over the process group (control plane only; the paper's ZeroMQ); returns this
    rank's arrivals.  No collective touches the step path."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [None]
    if rank == 0:
        obj = [route_trace(trace, world, sm, policy, max_batch, n_steps)]
    dist.broadcast_object_list(obj, src=0)
    return [a for a in trace if obj[0][a.rid] == rank]


# ---------------------------------------------------------------------------------------
# the GPU worker: real ig_edit_step steps on one device
# ---------------------------------------------------------------------------------------
class Engine:
    """One GPU worker (one process per GPU).  Runs a trace in real time: at every step
    boundary, arrived requests join the running batch while slots are free (continuous) or
    only when the batch is empty (static); one ig_edit_step per step; completions and joins
    are timed with device events.  One step is kept in flight so the copy lane's look-ahead
    crosses step boundaries."""

    def __init__(self, ig, ctx, desc, cache, sigmas, max_batch: int, stream, make_request):
        self.ig, self.ctx, self.d, self.cache, self.sig = ig, ctx, desc, cache, sigmas
        self.max_batch, self.stream, self.make_request = max_batch, stream, make_request
        self.n_steps = len(sigmas) - 1

    def run(self, trace: Sequence[Arrival], batching: str = "continuous"):
        import time
        import torch
        ig = self.ig
        pend = sorted(trace, key=lambda a: (a.t, a.rid))
        slots: List[Optional[dict]] = [None] * self.max_batch
        rec: Dict[int, list] = {}
        inflight = []  # (end_event, [(rid, finishing)])
        t0 = time.perf_counter()
        origin = torch.cuda.Event(enable_timing=True)
        origin.record(self.stream)
        i = 0
        steps = 0

        def now():
            return time.perf_counter() - t0

        while i < len(pend) or any(slots) or inflight:
            t = now()
            active = sum(1 for s in slots if s)
            if batching == "continuous" or active == 0:
                for k in range(self.max_batch):
                    if slots[k] is None and i < len(pend) and pend[i].t <= t:
                        a = pend[i]
                        i += 1
                        r = self.make_request(a)
                        r["step"] = 0
                        r["rid"] = a.rid
                        slots[k] = r
                        rec[a.rid] = [a.t, t, None]
            if not any(slots):
                if inflight:
                    self._retire(inflight.pop(0), origin, rec)
                    continue
                if i < len(pend):
                    time.sleep(max(0.0, min(pend[i].t - now(), 0.05)))
                continue
            reqs = [ig.make_req(k, s["latent"].data_ptr(), s["mask"], self.cache, s["step"],
                                float(self.sig[s["step"]]), float(self.sig[s["step"] + 1]),
                                s["txt"].data_ptr(), s["cond"].data_ptr())
                    for k, s in enumerate(slots) if s]
            ig.ig_edit_step(self.ctx, reqs, self.stream.cuda_stream)
            steps += 1
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(self.stream)
            done = []
            for k, s in enumerate(slots):
                if s:
                    s["step"] += 1
                    if s["step"] == self.n_steps:
                        done.append((s["rid"], s))
                        slots[k] = None
            inflight.append((ev, done))
            if len(inflight) > 1:
                self._retire(inflight.pop(0), origin, rec)
        wall = now()
        return rec, steps, wall

    def _retire(self, item, origin, rec):
        ev, done = item
        ev.synchronize()
        t_done = origin.elapsed_time(ev) * 1e-3
        for rid, s in done:
            rec[rid][2] = t_done
            if "free" in s:
                s["free"]()
