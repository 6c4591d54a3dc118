"""CPU tests of the multi-GPU host logic (§8(e)): OLS latency fits, Algorithm 1
(S:263-272 worked example), Algorithm 2 routing (argmin, lowest-id ties, slack, cost
monotonicity S:512-514), and the dispatcher over a world_size-2 gloo group."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import synth
from paper_2505_20600_b200 import placement as P


def test_fit_exact_line_and_degenerate():
    s, b, r2 = P.fit_ols([1, 2, 3], [2.5, 4.5, 6.5])
    assert abs(s - 2) < 1e-12 and abs(b - 0.5) < 1e-12 and abs(r2 - 1) < 1e-12
    s, b, r2 = P.fit_ols([1, 2, 3, 4], [1, 2, 3, 10])
    assert r2 < 1
    with pytest.raises(ValueError):
        P.fit_ols([2, 2, 2], [1, 2, 3])


def test_algorithm1_worked_example():
    # S:263 N=4, C_w=1, C_w/o=3, L=2 (SURVEY C-AMB 23, hand-checked)
    use, comp, load, t = P.algorithm1(4, 1.0, 3.0, 2.0, tie="<=")
    assert use == [True] * 4 and comp[1:] == [3, 5, 7, 9] and t == 9
    use, comp, load, t = P.algorithm1(4, 1.0, 3.0, 2.0, tie="<")
    assert use == [False, True, True, True] and comp[1:] == [3, 4, 5, 7] and t == 7
    plan, best = P.exact_plan(4, 1.0, 3.0, 2.0)
    assert best == 7


@pytest.mark.parametrize("N,cw,cwo,l", [(6, 1.0, 2.5, 1.7), (8, 0.4, 1.0, 0.9), (5, 2.0, 2.0, 0.1)])
def test_algorithm1_never_worse_than_all_compute_and_matches_pipeline(N, cw, cwo, l):
    use, comp, load, t = P.algorithm1(N, cw, cwo, l)
    assert t <= N * cwo + 1e-12
    assert abs(P.pipeline_latency(use, cw, cwo, l) - t) < 1e-9
    assert P.exact_plan(N, cw, cwo, l)[1] <= t + 1e-9


def _model():
    return P.LatencyModel(comp_slope=1 / 1.0e15, comp_intercept=1e-5, load_slope=1 / 5.0e10, load_intercept=2e-5)


def test_table1_work_matches_closed_form():
    d = synth.FLUX
    per_row = 2 * (3 * 3072 ** 2 + 3072 ** 2 + 2 * 3072 * 12288) + 4 * 4608 * 3072
    assert P.block_flops(d, 819) == per_row * (512 + 819)
    assert P.block_load_bytes(d, 819) == 2 * (4096 - 819) * 3072 * 2
    assert P.block_load_bytes(d, 0) == 0 and P.block_load_bytes(d, 4096) == 0


def _compute_bound():
    return P.LatencyModel(comp_slope=1 / 1.0e15, comp_intercept=1e-5, load_slope=1e-16, load_intercept=0.0)


def test_route_argmin_ties_and_slack():
    d = synth.FLUX
    pl = P.Placement(d, _model(), 3, max_batch=2)
    assert pl.route(500) == 0           # all empty: tie -> lowest id
    assert pl.route(500) == 1
    assert pl.route(500) == 2
    # SPEC S:488 derived example (compute-bound costs): A busy with m=0.8, B with m=0.1, new
    # m=0.3 -> B; a worker without slack is not a candidate
    pl = P.Placement(d, _compute_bound(), 3, max_batch=2)
    pl.workers[0].running = [int(0.8 * 4096)]
    pl.workers[1].running = [int(0.1 * 4096)]
    pl.workers[2].running = [10, 10]
    assert pl.route(int(0.3 * 4096)) == 1
    # every worker full -> global argmin over all of them
    pl = P.Placement(d, _compute_bound(), 2, max_batch=1)
    pl.workers[0].running = [3000]
    pl.workers[1].running = [200]
    assert pl.route(1000) == 1


def test_route_link_bound_pairs_small_with_large_masks():
    # over PCIe the K/V variant is link-bound for small m: joining a large-m (compute-heavy,
    # few cached bytes) batch is cheaper than joining a small-m (byte-heavy) batch
    d = synth.FLUX
    pl = P.Placement(d, _model(), 2, max_batch=4)
    pl.workers[0].running = [200, 200]
    pl.workers[1].running = [2400, 2400]
    assert pl.route(150) == 1


def test_route_cost_monotone_in_batch_membership():
    # adding a request to a worker's hypothetical batch never decreases calc_cost
    d = synth.FLUX
    for model in (_model(), _compute_bound()):
        pl = P.Placement(d, model, 1)
        for base in ([], [800], [800, 1200], [100, 3000, 2000]):
            for extra in (100, 1500, 4000):
                for n in (200, 2000):
                    assert pl.calc_cost(n, P.Worker(0, base + [extra])) >= pl.calc_cost(n, P.Worker(0, list(base))) - 1e-12


def test_route_balances_mixed_stream():
    d = synth.FLUX
    pl = P.Placement(d, _model(), 4, max_batch=8)
    import numpy as np
    rng = np.random.default_rng(0)
    for _ in range(24):
        pl.route(int(round(rng.uniform(0.05, 0.6) * 4096)))
    loads = [pl.batch_latency(w.running) for w in pl.workers]
    assert max(loads) <= 1.35 * min(loads)


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
    reqs = pl = None
    if rank == 0:
        reqs = [(i, 100 + 97 * i % 2400) for i in range(20)]
        pl = P.Placement(synth.FLUX, _model(), world, max_batch=16)
    mine = P.dispatch_gloo(reqs, pl)
    q.put((rank, mine))
    dist.barrier()
    dist.destroy_process_group()


def test_dispatch_gloo_world2():
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
    ids = sorted(i for r in got for i, _ in got[r])
    assert ids == list(range(20))                       # every request exactly once
    assert got[0] and got[1]                            # both replicas used


def test_uplink_term_steers_link_heavy_requests_off_a_loaded_uplink():
    """Workers 0 and 1 share one host uplink (as fast as ONE GPU's link), worker 2 has its own
    (SURVEY §8(e) uplink term).  Worker 0 already streams low-m (link-heavy) requests.  A new
    link-heavy request costs the same on the idle workers 1 and 2 without the uplink term (ties
    go to the lowest id: worker 1); with it, worker 1's loads would share worker 0's uplink, so
    Algorithm 2 picks worker 2."""
    m = _model()
    heavy = [120, 150, 100]  # n_m of ~3%: 97% of the K/V rows cross the link
    plain = P.Placement(synth.FLUX, m, 3, max_batch=8)
    aware = P.Placement(synth.FLUX, m, 3, max_batch=8, uplinks=[0, 0, 1], uplink_load_slope=m.load_slope)
    for pl in (plain, aware):
        pl.workers[0].running.extend(heavy)
    assert plain.route(130) == 1
    assert aware.route(130) == 2
    # the shared uplink binds: the sibling's predicted step is slower than the same batch alone
    assert aware.batch_latency([130], 1) > aware.batch_latency([130], 2)
