mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_unet_full.py -x -q -m gpu > gpurun_out/r3c25_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c25_tests.log
for v in gn0 gn1; do
  IG_LIB_OVERRIDE=ablibs/lib_$v.so timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:gn_apply --csv --log-file gpurun_out/r3c25_gn_$v.csv python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 --profile > /dev/null 2>&1; echo $v rc=$?
  python - <<P
import csv
rows=list(csv.reader(open("gpurun_out/r3c25_gn_$v.csv")))
hdr=None; t=0; n=0
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d["Metric Name"]=="gpu__time_duration.sum": t+=float(d["Metric Value"].replace(",","")); n+=1
print("$v gn_apply launches", n, "total us", t/1e3)
P
done
for v in gn0 gn1 gn0 gn1; do
  IG_LIB_OVERRIDE=ablibs/lib_$v.so timeout 600 python tools/unet_full_sweep.py --ms 0.2,1.0 --steps 4 --warmup 2 > gpurun_out/r3c25_sweep_$v.log 2>&1; echo $v rc=$?; grep '"m"' gpurun_out/r3c25_sweep_$v.log | head -2 | cut -c1-120
done
