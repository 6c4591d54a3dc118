"""Render one window of an IG_PROFILE_DUMP timeline (copy lane vs compute lane) as SVG and a
per-step summary: python tools/tl_svg.py dump.csv out.svg [t0_ms span_ms].

Records (ig_profile_read): kind,M,N,K,epi,ms,flops,bytes,start_ms; kind 6 = the copy lane's
cache copy of one block (M = block), every other kind a compute-stream launch (0 GEMM, 1
attention, 2 LN-mod, 3 qkv-post, 4 conditioning, 5 row kernels).  start_ms is relative to the
ig_profile_enable of the window (the last window in the file is drawn)."""
import sys

COL = {0: "#4c72b0", 1: "#dd8452", 2: "#55a868", 3: "#c44e52", 4: "#8172b3", 5: "#937860", 6: "#da8bc3"}
NAME = {0: "GEMM", 1: "attention", 2: "LN-mod", 3: "qkv-post", 4: "cond", 5: "rows", 6: "copy lane (block cache)"}
rows = [l.strip().split(",") for l in open(sys.argv[1]) if l.count(",") == 8]
wins, cur, last = [], [], -1.0
for r in rows:
    t = float(r[8])
    if cur and t < last - 200:
        wins.append(cur)
        cur, last = [], -1.0
    cur.append((int(r[0]), int(r[1]), float(r[5]), float(r[7]), t))
    last = max(last, t)
if cur:
    wins.append(cur)
recs = wins[-1]
t_end = max(r[4] + r[2] for r in recs)
t0 = float(sys.argv[3]) if len(sys.argv) > 3 else t_end * 0.4
span = float(sys.argv[4]) if len(sys.argv) > 4 else 250.0
sel = [r for r in recs if r[4] + r[2] > t0 and r[4] < t0 + span]
W, X0, H = 1400, 130, 40
sx = (W - X0 - 20) / span
out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="230" font-family="monospace" font-size="12">',
       f'<text x="10" y="18">libig lanes, {span:.0f} ms from t = {t0:.1f} ms (IG_PROFILE_DUMP, CUDA events per launch)</text>']
for lane, (lbl, y) in enumerate((("copy lane", 40), ("compute", 100))):
    out.append(f'<text x="10" y="{y + 25}">{lbl}</text>')
for k, b, ms, byt, t in sel:
    y = 40 if k == 6 else 100
    x = X0 + max(0.0, t - t0) * sx
    w = max(0.5, (min(t + ms, t0 + span) - max(t, t0)) * sx)
    out.append(f'<rect x="{x:.2f}" y="{y}" width="{w:.2f}" height="{H}" fill="{COL.get(k, "#999")}"><title>{NAME.get(k)} '
               f'block {b} {ms:.3f} ms</title></rect>')
for i in range(0, int(span) + 1, 25):
    x = X0 + i * sx
    out.append(f'<line x1="{x:.1f}" y1="150" x2="{x:.1f}" y2="155" stroke="black"/><text x="{x - 8:.1f}" y="168">{i}</text>')
lx = X0
for k in (0, 1, 2, 5, 6):
    out.append(f'<rect x="{lx}" y="190" width="12" height="12" fill="{COL[k]}"/><text x="{lx + 16}" y="201">{NAME[k]}</text>')
    lx += 40 + 8 * len(NAME[k])
out.append("</svg>")
open(sys.argv[2], "w").write("\n".join(out))
cp = [r for r in sel if r[0] == 6]
co = sorted([r for r in sel if r[0] != 6], key=lambda r: r[4])
busy_c = sum(min(r[4] + r[2], t0 + span) - max(r[4], t0) for r in cp)
busy_k, ce = 0.0, -1e9
for r in co:
    s, e = max(r[4], t0), min(r[4] + r[2], t0 + span)
    if e > ce:
        busy_k += e - max(s, ce)
        ce = e
print(f"window span {t_end:.1f} ms; drawn [{t0:.1f}, {t0 + span:.1f}] ms: copy lane busy {busy_c / span:.3f}, "
      f"compute lane busy {busy_k / span:.3f}, {len(cp)} block copies ({sum(r[3] for r in cp) / 1e9:.2f} GB), "
      f"{len(co)} compute launches")
