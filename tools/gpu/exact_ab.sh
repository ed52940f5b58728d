mkdir -p gpurun_out
python tools/gpu/exact_prof.py
REPS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/gpu/exact_prof.py 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
from collections import defaultdict
a=defaultdict(float)
for r in rows[1:]: a[r[ki].split('(')[0]]+=float(r[vi].replace(',',''))
for k,v in sorted(a.items(), key=lambda x:-x[1])[:6]: print(k[:50].ljust(50), round(v/1e6,2), 'ms')
"
timeout 900 python -m pytest tests/test_mask_gpu.py tests/test_select_ops_gpu.py tests/test_objective_gpu.py -x -q 2>&1 | tail -2
