"""Summarise ncu --set full captures (.ncu-rep) into a markdown block: duration, clocks, tensor
pipe, XU/FMA/ALU pipes, DRAM bytes, L2 hit rate, occupancy, registers / spills, and the top
warp-stall source lines.  Used for the profiles/r02_*.md evidence.

    python tools/ncu_summary.py gpurun_out/r2_gemm_full.ncu-rep [more.ncu-rep ...] > profiles/x.md
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    unit = dict(zip(h, units))
    return [dict(zip(h, r)) for r in rows[2:]], unit


def stalls(rep, top=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h = rows[1]
    try:
        isrc, iall = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        return []
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[iall] or 0), r[isrc].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    return [(100.0 * n / tot, s) for n, s in sorted(data, reverse=True)[:top]]


def main():
    for rep in sys.argv[1:]:
        print(f"### {rep}\n")
        launches, unit = raw(rep)
        for i, k in enumerate(launches):
            name = k.get("Kernel Name", "?")
            print(f"**launch {i}: `{name[:110]}`**\n")
            print("| metric | value |\n|---|---|")
            for m, label in WANT:
                v = k.get(m)
                if v is None:
                    continue
                print(f"| {label} | {v} {unit.get(m, '')} |")
            print()
        st = stalls(rep)
        if st:
            print("Top warp-stall samples by SASS instruction (all launches in the capture):\n")
            print("| % samples | instruction |\n|---|---|")
            for p, s in st:
                print(f"| {p:.1f} | `{s[:90]}` |")
            print()


if __name__ == "__main__":
    main()
