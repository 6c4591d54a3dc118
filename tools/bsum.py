"""Print the key numbers of bench.py JSON lines (files given on the command line)."""
import json
import sys

for fn in sys.argv[1:]:
    for line in open(fn):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        npl = d.get("no_plan_host_tier") or {}
        print(fn, "value", d.get("value"), "ms", d.get("ms_per_step"), "plan", d.get("plan", {}).get("k"),
              "link", d.get("host_link", {}).get("achieved_GBps"), "gemm", d.get("roofline", {}).get("achieved"),
              "attn", d.get("attn_roofline", {}).get("achieved"), "step_frac", d.get("step_roofline", {}).get("frac"),
              "noplan", npl.get("value"), npl.get("ms_per_step"), "clk", d.get("clocks", {}).get("sm_mhz"))
