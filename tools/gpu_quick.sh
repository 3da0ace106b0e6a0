# quick GPU iteration: parity tests then a short bench (args forwarded to bench.py)
python -m pytest tests -x -q -m gpu 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bq.json 2> gpurun_out/bq.err; echo bench_rc=$?
tail -4 gpurun_out/bq.err
python -c "
import json; d=json.load(open('gpurun_out/bq.json'))
print({k:d.get(k) for k in ['value','ms_per_step','e2e','roofline','per_query']})
print(d['config'].get('efS'), d['config'].get('recall'))"
