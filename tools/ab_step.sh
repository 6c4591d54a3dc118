#!/bin/bash
# Per-kernel-class time of one profiled Flux step (ncu, serialised) for several libig builds:
#   tools/ab_step.sh lib1 lib2 ...      (env passed through, e.g. KV_BLOCKS=37)
for lib in "$@"; do
  IG_LIB_OVERRIDE=$lib ncu --nvtx --nvtx-include "profile_step/" --metrics gpu__time_duration.sum --clock-control none \
    --csv python tools/step_profile.py 2>/dev/null | python -c "
import csv, sys, collections
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
h = rows[0]; ik = h.index('Kernel Name'); iv = h.index('Metric Value')
agg = collections.defaultdict(float)
for r in rows[1:]:
    agg[r[ik].split('(')[0].split('<')[0].replace('void ', '')] += float(r[iv].replace(',', ''))
print('$lib', ' '.join('%s=%.2fms' % (k.split('::')[-1], v / 1e6) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:4]))
"
done
