"""CPU tests of the serving loop's host logic: nearest-rank percentiles,
Poisson traces, the virtual-clock cluster simulation under step-level continuous vs static
batching, Algorithm-2 routing vs the request-/token-count baselines (P:690-695,
P:750-785), and trace dispatch over a world_size-2 gloo group."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth
from paper_2505_20600_b200 import placement as P
from paper_2505_20600_b200 import serve as S


def test_percentile_spec_examples():
    assert S.percentile(list(range(1, 11)), 0.95) == 10      # ceil(9.5) = 10th
    assert S.percentile([5], 0.5) == 5
    assert S.percentile([3, 1, 2], 1.0) == 3
    assert S.percentile([4, 1, 3, 2], 0.5) == 2               # ceil(2) = 2nd
    with pytest.raises(ValueError):
        S.percentile([], 0.5)
    with pytest.raises(ValueError):
        S.percentile([1.0], 0.0)


def test_poisson_trace_rate_and_determinism():
    a = S.poisson_trace(2.0, 4000, 4096, seed=3)
    b = S.poisson_trace(2.0, 4000, 4096, seed=3)
    assert [(x.t, x.n_m) for x in a] == [(x.t, x.n_m) for x in b]
    gaps = np.diff([0.0] + [x.t for x in a])
    assert abs(gaps.mean() - 0.5) < 0.03                       # mean inter-arrival 1/rate
    m = np.array([x.n_m for x in a]) / 4096
    assert m.min() >= 0.05 - 1e-3 and m.max() <= 0.60 + 1e-3 and abs(m.mean() - 0.325) < 0.01
    sk = np.array([x.n_m for x in S.poisson_trace(2.0, 4000, 4096, seed=3, skew="own")]) / 4096
    assert abs(sk.mean() - (0.05 + 0.55 / 9)) < 0.01           # Beta(1, 8) mean 1/9


def _sm(comp=1.0e15, load=5.0e10):
    return S.StepModel(synth.FLUX, P.LatencyModel(1 / comp, 1e-5, 1 / load, 2e-5))


def test_single_worker_continuous_batching_timeline():
    sm = _sm()
    trace = [S.Arrival(0, 0.0, 800), S.Arrival(1, 0.01, 1200), S.Arrival(2, 50.0, 400)]
    assign, rec = S.simulate_cluster(trace, 1, "mask_aware", sm, max_batch=8, n_steps=28)
    assert set(assign.values()) == {0}
    t1 = sm.step([800])
    # request 0 starts at once; request 1 joins at the next step boundary ("in just one step")
    assert rec[0][1] == 0.0 and abs(rec[1][1] - t1) < 1e-12
    for rid, (arr, adm, done) in rec.items():
        assert arr <= adm < done
        assert done - adm >= 28 * sm.step([trace[rid].n_m]) - 1e-9   # 28 steps of at least its own cost
    # the late request finds an idle worker: no queueing
    assert rec[2][1] == 50.0


def test_static_batching_waits_for_the_whole_batch():
    sm = _sm()
    trace = [S.Arrival(0, 0.0, 800), S.Arrival(1, 0.1, 1200)]
    _, rec_c = S.simulate_cluster(trace, 1, "mask_aware", sm, batching="continuous")
    _, rec_s = S.simulate_cluster(trace, 1, "mask_aware", sm, batching="static")
    assert abs(rec_s[1][1] - rec_s[0][2]) < 1e-12             # joins only when request 0 is done
    assert rec_c[1][2] < rec_s[1][2]                          # continuous finishes it earlier


def test_drain_cost_closed_form_and_monotone():
    sm = _sm()
    a = sm.drain_cost([(800, 28)])
    assert abs(a - 28 * sm.step([800])) < 1e-12
    b = sm.drain_cost([(800, 28), (1600, 10)])
    assert abs(b - (10 * sm.step([800, 1600]) + 18 * sm.step([800]))) < 1e-12
    assert b >= a


def test_mask_aware_routing_spec_example_and_balance():
    sm = _sm(load=1e30)  # compute-bound costs
    ws = [S.WorkerState(0), S.WorkerState(1)]
    ws[0].running = [[int(0.8 * 4096), 20, 100]]
    ws[1].running = [[int(0.1 * 4096), 20, 101]]
    assert S._route(ws, S.Arrival(5, 0.0, int(0.3 * 4096)), "mask_aware", sm, 8, 28) == 1
    # identical idle workers -> lowest id
    assert S._route([S.WorkerState(0), S.WorkerState(1)], S.Arrival(6, 0.0, 500), "mask_aware", sm, 8, 28) == 0
    # request-count baseline ignores mask sizes
    assert S._route(ws, S.Arrival(5, 0.0, 1000), "request_count", sm, 8, 28) == 0


@pytest.mark.parametrize("skew", [None, "public"])
def test_mask_aware_beats_request_count_on_p95(skew):
    # P:690-695 / SURVEY N3: on a mixed-mask Poisson trace at high load the mask-aware policy
    # gives a P95 latency no worse than request-count balancing
    sm = _sm()
    one = sm.step([1331] * 8) / 8 * 28          # ~ seconds of GPU work per request at batch 8
    trace = S.poisson_trace(4 * 0.8 / one, 160, 4096, seed=1, skew=skew)
    res = {}
    for pol in ("mask_aware", "request_count", "token_count"):
        _, rec = S.simulate_cluster(trace, 4, pol, sm)
        lat = [r[2] - r[0] for r in rec.values()]
        res[pol] = S.percentile(lat, 0.95)
    assert res["mask_aware"] <= res["request_count"] * 1.001
    assert all(v > 0 for v in res.values())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    trace = S.poisson_trace(3.0, 40, 4096, seed=5)
    mine = S.dispatch_trace(trace, _sm(), "mask_aware")
    q.put((rank, [a.rid for a in mine]))
    dist.barrier()
    dist.destroy_process_group()


def test_dispatch_trace_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(got[0] + got[1]) == list(range(40))
    assert got[0] and got[1]
