# dev helpers (source me): b = one bench.py line summarised (ms/step, per-level ms and iterations);
# cfg <c> = per-level device time of a BASELINE config (tools/run_config.py, second repetition)
b() { python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [(l['ms'], l['avg_iters']) for l in d['config']['per_level']])"; }
cfg() { python tools/run_config.py $1 2 2>&1 | grep "rep1 L" | python -c "
import sys, json
out=[]
for l in sys.stdin:
    d=json.loads(l[l.index('{'):]); out.append(f\"{l[5:7]} {d['ms_total']:.1f} ms ({d['avg_iters']:.0f} it)\")
print('config $1 total', round(sum(float(o.split()[1]) for o in out),1), 'ms:', '; '.join(out))"; }
