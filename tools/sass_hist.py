"""SASS opcode histogram of selected libig kernels (cuobjdump -sass): the evidence that the hot
kernels are tcgen05 (UTCHMMA / UTCBAR), TMEM (LDTM / STTM) and TMA (UTMALDG) code.

    python tools/sass_hist.py [paper_2505_20600_b200/lib/libig.so] > profiles/r02_sass_hist.md
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2505_20600_b200/lib/libig.so"
KERNELS = {"gemm_tc2_kernel": "gemm_tc2_kernel", "gemm_tc_kernel<256, false>": "gemm_tc_kernelILi256ELb0E",
           "gemm_tc_kernel<256, true> (implicit conv)": "gemm_tc_kernelILi256ELb1E",
           "attn_tc_kernel<128>": "attn_tc_kernelILi128E", "attn_tc_kernel<64>": "attn_tc_kernelILi64E"}
KEY = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMAPF", "SYNCS", "MUFU", "FFMA", "FFMA2", "FADD2", "FMUL2",
       "FMNMX", "FMNMX3", "HMMA", "LDG", "STG", "LDS", "STS", "BAR"]

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
print(f"SASS opcode counts (static instructions) in `{LIB}`, `cuobjdump -sass`.\n")
print("| kernel | " + " | ".join(KEY) + " |")
print("|---|" + "---|" * len(KEY))
for label, pat in KERNELS.items():
    body = next((f for f in funcs if pat in f.split("\n", 1)[0]), None)
    if body is None:
        continue
    ops = collections.Counter()
    for line in body.split("\n"):
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
        if m:
            ops[m.group(1)] += 1
    print(f"| {label} | " + " | ".join(str(ops.get(k, 0)) for k in KEY) + " |")
