"""Analyse an IG_PROFILE_DUMP timeline (kind,M,N,K,epi,ms,flops,bytes,start_ms per record;
kind 6 = copy-lane block copy, M = block): copy-lane busy time, its idle gaps, and the
compute-lane busy time, per profiled window (start_ms restarts at each ig_profile_enable)."""
import sys

rows = [l.strip().split(",") for l in open(sys.argv[1]) if l.count(",") == 8]
wins, cur, last = [], [], -1.0
for r in rows:
    t = float(r[8])
    if cur and t < last - 200:  # the time origin moved: a new window
        wins.append(cur)
        cur, last = [], -1.0
    cur.append((int(r[0]), int(r[1]), float(r[5]), float(r[7]), t))
    last = max(last, t)
if cur:
    wins.append(cur)
for w, recs in enumerate(wins):
    cp = sorted([r for r in recs if r[0] == 6], key=lambda r: r[4])
    co = sorted([r for r in recs if r[0] != 6], key=lambda r: r[4])
    t_end = max(r[4] + r[2] for r in recs)
    busy_c = sum(r[2] for r in cp)
    gaps = [(cp[i][4] - (cp[i - 1][4] + cp[i - 1][2]), cp[i][1], cp[i - 1][1]) for i in range(1, len(cp))]
    big = sorted([g for g in gaps if g[0] > 0.5], reverse=True)[:12]
    # compute union
    busy_k, ce = 0.0, -1e9
    for r in co:
        s, e = r[4], r[4] + r[2]
        if e > ce:
            busy_k += e - max(s, ce)
            ce = e
    print(f"window {w}: span {t_end:.1f} ms  copy busy {busy_c:.1f} ms ({len(cp)} copies, "
          f"{sum(r[3] for r in cp) / 1e9:.2f} GB)  compute busy {busy_k:.1f} ms")
    print("  largest copy-lane gaps (ms, block, after block):", [(round(g, 2), b, a) for g, b, a in big])
