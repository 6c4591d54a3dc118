"""Build libig.so in-tree with nvcc for sm_100a (B200).  Used by __graft_entry__.build().

    python -m paper_2505_20600_b200.build [--debug] [--out PATH] [--define NAME[=VAL]]...
"""
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "lib", "libig.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-Xptxas", "-v"]


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _objdir(extra):
    if not extra:
        return OBJ
    import hashlib
    return OBJ + "_" + hashlib.sha1(" ".join(extra).encode()).hexdigest()[:10]


def _compile(src, extra):
    obj = os.path.join(_objdir(extra), src[:-3] + ".o")
    cmd = [NVCC] + ARCH + FLAGS + extra + ["-c", os.path.join(CSRC, src), "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, p.returncode, p.stdout + p.stderr


def build(verbose=False, extra=(), out=None):
    os.makedirs(_objdir(list(extra)), exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    extra = list(extra)
    objs, logs = [], {}
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for src, obj, rc, log in ex.map(lambda s: _compile(s, extra), sources()):
            logs[src] = log
            if rc != 0:
                raise RuntimeError(f"nvcc failed on {src}:\n{log}")
            objs.append(obj)
    lib = out or LIB
    link = [NVCC] + ARCH + ["-shared", "--cudart", "static", "-o", lib] + objs
    p = subprocess.run(link, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError("link failed:\n" + p.stdout + p.stderr)
    with open(os.path.join(ROOT, "build", "ptxas.log"), "w") as f:
        for k, v in logs.items():
            f.write(f"==== {k}\n{v}\n")
    if verbose:
        for k, v in logs.items():
            print(f"==== {k}\n{v}")
    return lib


if __name__ == "__main__":
    ex = []
    if "--debug" in sys.argv:
        ex.append("-G")
    if "--hang-check" in sys.argv:
        ex.append("-DIG_HANG_CHECK")
    out = None
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
    for i, a in enumerate(sys.argv):  # A/B variants: --define NAME[=VALUE] (repeatable)
        if a == "--define":
            ex.append("-D" + sys.argv[i + 1])
    print(build(verbose="-v" in sys.argv, extra=ex, out=out))
