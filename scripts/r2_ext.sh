#!/bin/bash
# EXT prime-length passes: parity (small + Duke head grid), then timing at duke_head and head_1mm
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ext_prime" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "duke" -s 2>&1 | grep -E "rel l2|passed|failed|Error" | tail -3
Q="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
for c in duke_head head_1mm; do
timeout 300 $Q --config $c > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err
python -c "
import json; d=json.loads(open('gpurun_out/q_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],3), d['stage_ms'], {k: round(v.get('ms_per_step',0),3) for k, v in d['strategies'].items()})" || tail -5 gpurun_out/q_$c.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/duke_launches.csv $Q --steps 1 --warmup 1 --config duke_head > /dev/null 2>&1
python - <<'PY'
import csv, collections
t = collections.defaultdict(float); n = collections.Counter()
rows = list(csv.reader(open('gpurun_out/duke_launches.csv')))
hdr = None
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            k = d['Kernel Name'].split('(')[0][:60]; t[k] += float(d['Metric Value']); n[k] += 1
for k, v in sorted(t.items(), key=lambda x: -x[1])[:14]: print(f"{v/1e6:9.3f} ms {n[k]:4d} {k}")
PY
