set -x
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q 2>&1 | tail -5
timeout 300 python scripts/probes/bwd_probe.py 2>&1 | tail -4
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bwd|unpool" --csv --log-file gpurun_out/bwd_launch.csv python scripts/probes/bwd_probe.py > /dev/null 2>&1
python - <<'P'
import csv,collections
d=collections.defaultdict(list)
for r in csv.DictReader(l for l in open('gpurun_out/bwd_launch.csv') if l.startswith('"')):
    if r['Metric Name']=='gpu__time_duration.sum': d[r['Kernel Name'][:40]].append(float(r['Metric Value'].replace(',','')))
for k,v in d.items(): print(k,len(v),sum(v)/len(v)/1e6,'ms')
P
