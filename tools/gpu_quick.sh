timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/gputests_q.log 2>&1; echo tests rc=$?
grep -E "passed|failed|error" gpurun_out/gputests_q.log | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
python - <<'PY'
import json; d=json.loads(open('gpurun_out/bench_q.json').read())
print('C2', round(d['value'],1), round(d['roofline']['frac'],4), 'probe', round(d['roofline']['write_probe_gbs']), d['clocks'])
for k,v in d['configs'].items():
    if 'roofline' in v: print(k, round(v['value'],1), round(v['roofline']['frac'],4))
    elif 'value' in v: print(k, round(v['value'],1), v.get('unit'))
    else: print(k, {kk: round(vv['value'],1) for kk,vv in v.items()})
PY
