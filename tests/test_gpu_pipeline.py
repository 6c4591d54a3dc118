"""GPU tests of the bench's own workload shape and of the two-lane pipeline:

* the continuous-batching schedule bench.py times — members at different denoising steps and
  sigmas, a member leaving and a new request joining the same slot mid-run (P:642-659 step-level
  continuous batching), a host-tier hybrid K/V + Y cache prefetched with a ring at least as deep
  as the step, the Algorithm-1 plan chosen per step by the latency model
   — replayed request by request through the float64 oracle (C-TOL 2e-2);
* race tests: NaN-poisoned ring buffers between steps (every row a step reads must be staged in
  that step: RAW), a slow copy lane and a slow compute lane (bitwise equal to the normal run),
  and negative controls that drop the RAW or the WAR event and must change the result;
* fault injection: a corrupted cached row must turn parity red;
* batch invariance across the GEMM tile-path switch (2-CTA 256x256, 1-CTA 128x256 and 128x128
  tiles chosen by problem size, SURVEY §8(c) requirement 1): rows computed in a small-M GEMM are
  bitwise equal to the same rows inside a large-M GEMM;
* ig_mask_build_host (admission without a device sync) equals ig_mask_build bit for bit;
  ig_debug_dump_kv returns the merged positional K/V buffer (fresh rows + cached rows).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2505_20600_b200 import ig
from gpu_util import Model, Request, ctol, fill_cache, hybrid_planes

pytestmark = pytest.mark.gpu

D = synth.FLUX_SMALL
N_SCHED = 6  # denoising steps of the schedule (bench: 28)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


class Member:
    """One request of the continuous batch: inputs, its mask handle and its step history."""

    def __init__(self, m, rid, mask_np, host_mask=False, stream=0):
        self.rid = rid
        self.latent = synth.make_latent(D, rid).cuda()
        self.latent0 = self.latent.clone()
        self.txt = synth.make_txt(D, rid, "cpu", torch.bfloat16).cuda()
        self.cond = synth.make_cond(D, rid).cuda()
        self.mask_np = mask_np.astype(np.uint8)
        if host_mask:
            self.mask, self.n_m = ig.ig_mask_build_host(m.ctx, self.mask_np, stream)
        else:
            self.mask_dev = torch.from_numpy(self.mask_np).cuda()
            self.mask, self.n_m = ig.ig_mask_build(m.ctx, self.mask_dev.data_ptr(), 0)
        self.step = 0
        self.log = []  # (step, plan k) of every batch step it took part in

    def req(self, slot, cache, sig):
        return ig.make_req(slot, self.latent.data_ptr(), self.mask, cache, self.step, float(sig[self.step]),
                           float(sig[self.step + 1]), self.txt.data_ptr(), self.cond.data_ptr())


def _mask(rid):
    rng = np.random.default_rng(7919 * rid + 5)
    n = int(round(rng.uniform(0.05, 0.6) * D.L_img))
    return synth.rect_mask_count(D, n, rng) if rid % 2 == 0 else synth.blob_mask_count(D, n, rng)


def _setup(kind, depth, max_batch=4):
    """ctx + host-tier cache of N_SCHED steps: kind 'hybrid' (2 K/V + 2 Y blocks, interleaved)
    or 'kv'.  Returns (model, cache, host copies for the oracle)."""
    y = kind == "hybrid"
    m = Model(D, ig.IG_BF16, opts=ig.ig_ctx_opts(max_batch, 0, depth, 1, 0, 0, int(y), 2 if y else 0))
    kv = synth.make_cache_kv(D, 30, N_SCHED, dtype=torch.bfloat16)
    yv = synth.make_cache_y(D, 30, N_SCHED, dtype=torch.bfloat16)
    tlat = torch.stack([synth.make_latent(D, 1100 + s) for s in range(N_SCHED)])
    ym = set(ig.y_block_modes(D.n_blocks, 2)) if y else None
    cache = ig.ig_cache_create(m.ctx, N_SCHED, ig.IG_CACHE_HOST)
    fill_cache(m, cache, hybrid_planes(kv, yv, ym) if y else kv, tlat)
    host = (kv.double().numpy(), yv.double().numpy(), tlat.double().numpy(), ym)
    return m, cache, host


def _run(m, cache, n_batch_steps, rid0=300, stream=None, between=None, host_masks=True):
    """The bench's schedule on max_batch slots: slot i starts at step i*N/B; a member that
    finishes its last step leaves and a new request joins the same slot at the next step.
    Returns every member (finished or not) in admission order."""
    sig = synth.flow_sigmas(N_SCHED)
    mb = m_slots = 4
    st = stream.cuda_stream if stream is not None else 0
    members, slots = [], []
    nxt = rid0
    for i in range(m_slots):
        mem = Member(m, nxt, _mask(nxt), host_mask=host_masks, stream=st)
        mem.step = (i * N_SCHED) // mb
        nxt += 1
        members.append(mem)
        slots.append(mem)
    for t in range(n_batch_steps):
        if between is not None:
            between(t)
        ig.ig_edit_step(m.ctx, [r.req(i, cache, sig) for i, r in enumerate(slots)], st)
        k = ig.ig_last_plan(m.ctx)
        for i, r in enumerate(slots):
            r.log.append((r.step, k))
            r.step += 1
            if r.step == N_SCHED:  # leaves; a new request joins this slot
                mem = Member(m, nxt, _mask(nxt), host_mask=host_masks, stream=st)
                nxt += 1
                members.append(mem)
                slots[i] = mem
    torch.cuda.synchronize()
    return members


def _oracle_replay(W, mem, host, kind):
    kv, yv, tlat, ym = host
    sig = synth.flow_sigmas(N_SCHED)
    lat0 = mem.latent0.double().cpu().numpy()
    txt = mem.txt.cpu().double().numpy()
    cond = mem.cond.cpu().double().numpy()
    x = lat0
    for s, k in mem.log:
        if kind == "hybrid":
            x = oracle.edit_step_y(D, W, x, mem.mask_np, yv[s], tlat[s], sig[s], sig[s + 1], txt, cond, k=k,
                                   y_blocks=ym, kv_cache_step=kv[s])
        else:
            x = oracle.edit_step_planned(D, W, x, mem.mask_np, kv[s], tlat[s], k, sig[s], sig[s + 1], txt, cond)
    return x


def _free(m, cache, members):
    for r in members:
        ig.ig_mask_free(r.mask)
    ig.ig_cache_free(cache)
    m.close()


# ------------------------------------------------------------------ the bench's workload shape
@pytest.mark.parametrize("kind,depth,plan", [("hybrid", 4, "model"), ("hybrid", 8, "k1"), ("kv", 2, "model"),
                                             ("kv", 4, "none")])
def test_staggered_continuous_batch_vs_oracle(kind, depth, plan):
    """8 batch steps of the staggered schedule (members at 4 different steps and sigmas, 3+
    leave/join events in reused slots), host-tier cache, copy lane ring depth >= blocks for the
    first two cases; every member replayed through the oracle with the plan k the GPU chose."""
    m, cache, host = _setup(kind, depth)
    if plan == "model":  # slow link vs fast compute: the planner buys a dense prefix on some steps
        ig.ig_set_plan(m.ctx, 2, 0, 1.0 / 1e14, 2e-6, 1.0 / 2e9, 1e-6)
    elif plan == "k1":
        ig.ig_set_plan(m.ctx, 1, 1)
    stream = torch.cuda.Stream()
    members = _run(m, cache, 8, stream=stream)
    assert len(members) >= 7  # at least three joins
    ks = {k for r in members for _, k in r.log}
    if plan == "model":
        print("plan k per step:", sorted(ks))
    W = m.host_weights()
    for r in members:
        ref = _oracle_replay(W, r, host, kind)
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, ref, 2e-2)
        assert ok, (r.rid, r.log, worst)
        un = r.mask_np == 0
        assert np.array_equal(got[un], r.latent0.double().cpu().numpy()[un])
    _free(m, cache, members)


def test_staggered_plan_model_uses_a_prefix():
    """The latency model of the parametrised run above does pick dense prefixes (k > 0) on this
    schedule, so the planned path is really exercised against the oracle."""
    m, cache, _ = _setup("hybrid", 4)
    ig.ig_set_plan(m.ctx, 2, 0, 1.0 / 1e14, 2e-6, 1.0 / 2e9, 1e-6)
    members = _run(m, cache, 4)
    assert max(k for r in members for _, k in r.log) > 0
    _free(m, cache, members)


# ------------------------------------------------------------------ race tests (T5)
def _latents(members):
    return {r.rid: r.latent.clone() for r in members}


def _scenario(kind, depth, dbg=(), poison=False, steps=5, plan=None):
    m, cache, host = _setup(kind, depth)
    if plan:
        ig.ig_set_plan(m.ctx, 1, plan)
    for key, val in dbg:
        ig.ig_debug_set(m.ctx, key, val)

    def between(t):
        if poison:
            torch.cuda.synchronize()
            ig.ig_debug_set(m.ctx, ig.IG_DBG_POISON_RING, 1)

    members = _run(m, cache, steps, between=between)
    out = _latents(members)
    W = m.host_weights()
    return m, cache, host, members, out, W


def _same(a, b):
    return all(torch.equal(a[k], b[k]) for k in a)


@pytest.mark.parametrize("kind,depth", [("hybrid", 4), ("kv", 1)])
def test_poison_and_slow_lanes_are_invisible(kind, depth):
    """NaN-poisoning every ring buffer before each step, a copy lane slowed by 300 us per block and
    a compute lane slowed by 300 us before each attention all leave the result bitwise unchanged
    (every row a step reads is staged in that step; RAW and WAR events order the lanes)."""
    runs = []
    for dbg, poison in (((), False), ((), True), (((ig.IG_DBG_SPIN_COPY_NS, 300_000),), True),
                        (((ig.IG_DBG_SPIN_COMPUTE_NS, 300_000),), False)):
        m, cache, _, members, out, _ = _scenario(kind, depth, dbg, poison)
        runs.append(out)
        _free(m, cache, members)
    for i in range(1, len(runs)):
        assert _same(runs[0], runs[i]), i
    assert all(torch.isfinite(v).all() for v in runs[1].values())


def test_dropped_raw_wait_is_detected():
    """Negative control: without the RAW wait (compute does not wait for the block's copy), a
    slow copy lane and a poisoned ring make attention read NaN rows."""
    m, cache, _, members, out, _ = _scenario("kv", 2, ((ig.IG_DBG_DROP_RAW, 1), (ig.IG_DBG_SPIN_COPY_NS, 2_000_000)),
                                             poison=True, steps=2)
    assert not all(torch.isfinite(v).all() for v in out.values())
    _free(m, cache, members)


def test_dropped_war_wait_is_detected():
    """Negative control: without the WAR wait the copy of block b + R overwrites ring buffer
    b % R while a slowed compute lane has not yet run block b's attention (depth 1, R = 2 < 4
    blocks), so the result changes."""
    m, cache, _, members, ref, _ = _scenario("kv", 1, steps=2)
    _free(m, cache, members)
    m, cache, _, members, bad, _ = _scenario("kv", 1, ((ig.IG_DBG_DROP_WAR, 1), (ig.IG_DBG_SPIN_COMPUTE_NS, 3_000_000)),
                                             steps=2)
    assert not _same(ref, bad)
    _free(m, cache, members)


def test_corrupted_cache_row_turns_parity_red():
    """Fault injection: +32 on every element of one staged cached K/V row per block.
    The same scenario that passes parity without the fault must fail it with the fault."""
    for corrupt in (0, 32):
        m, cache, host, members, out, W = _scenario("kv", 2, ((ig.IG_DBG_CORRUPT_ROW, corrupt),), steps=2)
        oks = []
        for r in members:
            if not r.log:
                continue
            ref = _oracle_replay(W, r, host, "kv")
            oks.append(ctol(r.latent.double().cpu().numpy(), ref, 2e-2)[0])
        if corrupt:
            assert not all(oks)
        else:
            assert all(oks)
        _free(m, cache, members)


# ------------------------------------------------------------------ boundary helpers
def test_mask_build_host_equals_device_build():
    m = Model(D, ig.IG_BF16, opts=ig.ig_ctx_opts(2, 0, 2, 1, 0))
    for rid in range(6):
        mk = _mask(rid)
        if rid == 4:
            mk = np.zeros(D.L_img, np.uint8)
        if rid == 5:
            mk = np.ones(D.L_img, np.uint8)
        dev = torch.from_numpy(mk).cuda()
        a, na = ig.ig_mask_build(m.ctx, dev.data_ptr(), 0)
        b, nb = ig.ig_mask_build_host(m.ctx, mk, 0)
        torch.cuda.synchronize()
        assert na == nb == int(mk.sum())
        out = []
        for h in (a, b):
            pm, pu, n = ig.ig_mask_indices(h)
            buf = torch.empty(2 * D.L_img, dtype=torch.int32, device="cuda")
            ig.ig_copy(buf.data_ptr(), pm, 2 * D.L_img * 4)
            out.append(buf.cpu().numpy())
        assert np.array_equal(out[0][:na], np.flatnonzero(mk))
        assert np.array_equal(out[0][D.L_img:2 * D.L_img - na], np.flatnonzero(mk == 0))
        assert np.array_equal(out[0][:na], out[1][:na])
        assert np.array_equal(out[0][D.L_img:2 * D.L_img - na], out[1][D.L_img:2 * D.L_img - na])
        ig.ig_mask_free(a)
        ig.ig_mask_free(b)
    m.close()


def test_debug_dump_kv_is_the_positional_merge():
    """After a one-request step (depth 4 >= blocks, so every block's ring buffer survives), the
    dumped buffer of block b holds the cached K/V rows at the unmasked positions L_txt + i
    (bitwise: pure copies) and finite fresh rows at the masked positions."""
    m, cache, host = _setup("kv", 4)
    kv = host[0]
    mem = Member(m, 77, _mask(77))
    sig = synth.flow_sigmas(N_SCHED)
    ig.ig_edit_step(m.ctx, [mem.req(1, cache, sig)], 0)
    torch.cuda.synchronize()
    L, H = D.L, D.hidden
    un = np.flatnonzero(mem.mask_np == 0)
    mk = np.flatnonzero(mem.mask_np)
    for b in range(D.n_blocks):
        k = torch.empty(L, H, dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        ig.ig_debug_dump_kv(m.ctx, 1, b, k.data_ptr(), v.data_ptr())
        kh, vh = k.double().cpu().numpy(), v.double().cpu().numpy()
        assert np.array_equal(kh[D.txt_len + un], kv[0, b, 0][un])
        assert np.array_equal(vh[D.txt_len + un], kv[0, b, 1][un])
        assert np.isfinite(kh[D.txt_len + mk]).all() and np.isfinite(kh[:D.txt_len]).all()
    ig.ig_mask_free(mem.mask)
    ig.ig_cache_free(cache)
    m.close()


@pytest.mark.parametrize("M_small,N,K,epi,M_big", [(300, 3072, 3072, 0, 14720), (100, 21504, 3072, 1, 14720),
                                                  (700, 3072, 12288, 2, 14720), (60, 9216, 3072, 0, 14720),
                                                  (300, 1280, 1280, 0, 8192), (700, 1280, 5120, 2, 8192),
                                                  (1000, 640, 640, 1, 32768), (449, 1536, 6144, 2, 14720),
                                                  (300, 1536, 1536, 0, 8192)])
def test_gemm_rows_bitwise_across_tile_paths(M_small, N, K, epi, M_big):
    """The same A rows through a small-M GEMM (1-CTA 128x128 tiles when the 2-CTA grid would be
    under SMs/4, 128x64 tiles when even those are under SMs/2 — the single-request SD3 shapes —
    or 128x256 tiles at M <= 128) and inside a large-M GEMM (2-CTA 256x256 tiles) give bitwise
    equal outputs: every output is one full-K accumulation in the same K order."""
    g = torch.Generator(device="cuda").manual_seed(N + K + epi)
    A = (torch.randn(M_big, K, device="cuda", generator=g) / 4).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g).bfloat16()
    if epi == 2:  # fp32 gated residual
        gate = torch.rand(N, device="cuda", generator=g)
        X0 = torch.randn(M_big, N, device="cuda", generator=g)
        Xb, Xs = X0.clone(), X0[:M_small].clone()
        ig.ig_op_gemm_gated(ig.IG_BF16, A.data_ptr(), K, B.data_ptr(), K, bias.data_ptr(), Xb.data_ptr(), N,
                            gate.data_ptr(), M_big, N, K)
        ig.ig_op_gemm_gated(ig.IG_BF16, A.data_ptr(), K, B.data_ptr(), K, bias.data_ptr(), Xs.data_ptr(), N,
                            gate.data_ptr(), M_small, N, K)
        torch.cuda.synchronize()
        assert torch.equal(Xb[:M_small], Xs)
    else:
        Cb = torch.empty(M_big, N, device="cuda", dtype=torch.bfloat16)
        Cs = torch.empty(M_small, N, device="cuda", dtype=torch.bfloat16)
        ig.ig_op_gemm(ig.IG_BF16, A.data_ptr(), K, B.data_ptr(), K, bias.data_ptr(), Cb.data_ptr(), N, M_big, N, K, epi)
        ig.ig_op_gemm(ig.IG_BF16, A.data_ptr(), K, B.data_ptr(), K, bias.data_ptr(), Cs.data_ptr(), N, M_small, N, K, epi)
        torch.cuda.synchronize()
        assert torch.equal(Cb[:M_small], Cs)
        ref = (A[:M_small].float() @ B.float().t() + bias.float())
        if epi == 1:
            ref = torch.nn.functional.gelu(ref, approximate="tanh")
        assert torch.allclose(Cs.float(), ref, rtol=2e-2, atol=2e-2 * ref.pow(2).mean().sqrt().item())


# ------------------------------------------------------------------ peer-HBM template pool (N4)
def _ipc_child(handle, q):
    import sys as _s
    import os as _o
    _s.path.insert(0, _o.path.dirname(_o.path.abspath(__file__)))
    import torch as _t
    import synth as _sy
    from paper_2505_20600_b200 import ig as _ig
    from gpu_util import Model as _M
    _t.cuda.set_device(0)
    m = _M(D, _ig.IG_BF16, opts=_ig.ig_ctx_opts(4, 0, 2, 1, 0))
    cache = _ig.ig_cache_import(m.ctx, handle)
    mem = Member(m, 91, _mask(91))
    sig = _sy.flow_sigmas(N_SCHED)
    mem.step = 2
    _ig.ig_edit_step(m.ctx, [mem.req(0, cache, sig)], 0)
    _t.cuda.synchronize()
    q.put(mem.latent.cpu().numpy().tobytes())
    _ig.ig_cache_free(cache)
    _ig.ig_mask_free(mem.mask)
    m.close()


def test_peer_pool_cache_import_in_another_process():
    """A device-tier cache exported by this process (CUDA IPC) and imported by a second process
    (here on the same GPU; across GPUs the copy lane's gather then reads the owner's HBM over
    NVLink): the importer's edit step equals the owner's on its own cache, bit for bit."""
    import multiprocessing as mp
    m = Model(D, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0))
    kv = synth.make_cache_kv(D, 30, N_SCHED, dtype=torch.bfloat16)
    tlat = torch.stack([synth.make_latent(D, 1100 + s) for s in range(N_SCHED)])
    cache = ig.ig_cache_create(m.ctx, N_SCHED, ig.IG_CACHE_DEVICE)
    fill_cache(m, cache, kv, tlat)
    handle = ig.ig_cache_export(cache)
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    p = ctx_mp.Process(target=_ipc_child, args=(handle, q))
    p.start()
    got = q.get(timeout=300)
    p.join(timeout=120)
    assert p.exitcode == 0
    mem = Member(m, 91, _mask(91))
    mem.step = 2
    ig.ig_edit_step(m.ctx, [mem.req(0, cache, synth.flow_sigmas(N_SCHED))], 0)
    torch.cuda.synchronize()
    assert mem.latent.cpu().numpy().tobytes() == got
    assert not torch.equal(mem.latent, mem.latent0)
    ig.ig_mask_free(mem.mask)
    ig.ig_cache_free(cache)
    m.close()
