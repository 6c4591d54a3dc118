"""Copy-engine probe for the copy lane (a7): host enqueue cost per call and achieved host-link
GB/s of many small pinned H2D cudaMemcpyAsync calls vs strided cudaMemcpy2DAsync calls.
Prints one JSON object.  (One GPU; run under gpurun.)"""
import ctypes, json, time, os, glob
import torch

cands = sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))
rt = ctypes.CDLL(cands[0])
vp, sz = ctypes.c_void_p, ctypes.c_size_t
rt.cudaMemcpyAsync.argtypes = [vp, vp, sz, ctypes.c_int, vp]
rt.cudaMemcpy2DAsync.argtypes = [vp, sz, vp, sz, sz, sz, ctypes.c_int, vp]
torch.cuda.init()
dev = torch.device("cuda:0")
NB = 1 << 30
h = torch.empty(NB, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(NB, dtype=torch.uint8, device=dev)
st = torch.cuda.Stream()
sp = st.cuda_stream
out = {}


def run(label, calls):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(st):
        e0.record(st)
        t0 = time.perf_counter()
        nbytes = 0
        for c in calls:
            nbytes += c()
        t1 = time.perf_counter()
        e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out[label] = {"calls": len(calls), "host_us_per_call": round((t1 - t0) / len(calls) * 1e6, 2),
                  "gpu_ms": round(ms, 3), "GBps": round(nbytes / ms / 1e6, 2)}


hp, dp = h.data_ptr(), d.data_ptr()
for row_kb in (6, 24, 96, 384, 1536):
    b = row_kb * 1024
    n = min(4000, NB // b)
    def mk(i, b=b):
        def c():
            rt.cudaMemcpyAsync(dp + i * b, hp + i * b, b, 4, sp)
            return b
        return c
    run(f"1d_{row_kb}KB", [mk(i) for i in range(n)])
# 2D: `height` runs of `width` bytes one image row (64 tokens x 6 KB) apart
pitch = 64 * 6144
for wt, ht in ((30, 30), (50, 40), (10, 64), (4, 64)):
    w = wt * 6144
    n = min(400, NB // (pitch * ht))
    def mk2(i, w=w, ht=ht):
        def c():
            off = i * pitch * ht
            rt.cudaMemcpy2DAsync(dp + off, pitch, hp + off, pitch, w, ht, 4, sp)
            return w * ht
        return c
    run(f"2d_{wt}tok_x{ht}", [mk2(i) for i in range(n)])
# 3-D: the K and V planes of one group in ONE call (depth 2), spans and strided rows
class PP(ctypes.Structure):
    _fields_ = [("ptr", vp), ("pitch", sz), ("xsize", sz), ("ysize", sz)]
class Pos(ctypes.Structure):
    _fields_ = [("x", sz), ("y", sz), ("z", sz)]
class Ext(ctypes.Structure):
    _fields_ = [("width", sz), ("height", sz), ("depth", sz)]
class P3(ctypes.Structure):
    _fields_ = [("srcArray", vp), ("srcPos", Pos), ("srcPtr", PP), ("dstArray", vp), ("dstPos", Pos),
                ("dstPtr", PP), ("extent", Ext), ("kind", ctypes.c_int)]
rt.cudaMemcpy3DAsync.argtypes = [ctypes.POINTER(P3), vp]
splane, dplane = 4096 * 6144, 4608 * 6144
for wt, ht in ((1, 1), (8, 1), (64, 1), (30, 30), (4, 64)):
    w = wt * 6144
    span = ht == 1
    n = min(300, NB // (2 * dplane + pitch * ht) // 1)
    def mk3(i, w=w, ht=ht, span=span):
        def c():
            p3 = P3()
            off = (i % 8) * pitch * 2
            sp_, dp_ = (splane, dplane) if span else (pitch, pitch)
            p3.srcPtr = PP(hp + off, sp_, w, splane // sp_)
            p3.dstPtr = PP(dp + off, dp_, w, dplane // dp_)
            p3.extent = Ext(w, ht, 2)
            p3.kind = 4
            e = rt.cudaMemcpy3DAsync(ctypes.byref(p3), sp)
            assert e == 0, e
            return 2 * w * ht
        return c
    run(f"3d_kv_{wt}tok_x{ht}", [mk3(i) for i in range(n)])
# one big copy: the link's ceiling
run("1d_512MB", [lambda: (rt.cudaMemcpyAsync(dp, hp, 512 << 20, 4, sp), 512 << 20)[1]])
print(json.dumps(out))
