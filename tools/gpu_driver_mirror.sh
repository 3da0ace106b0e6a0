# What the driver runs at round end, on one B200: GPU tests, smoke, the reference arm, the default bench line
R=gpurun_out/mirror; mkdir -p $R
timeout 1500 python -m pytest tests -x -q -m gpu > $R/pytest_gpu.txt 2>&1; echo pytest=$?; tail -2 $R/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.txt 2>&1; echo smoke=$?; tail -1 $R/smoke.txt
timeout 900 python bench.py --impl reference > $R/ref.json 2> $R/ref.err; echo ref=$?
timeout 900 python bench.py > $R/bench.json 2> $R/bench.err; echo bench=$?
python -c "
import json
a=json.load(open('$R/bench.json')); b=json.load(open('$R/ref.json'))
print('value', a['value'], 'e2e', a['e2e']['value'], 'frac', a['roofline']['frac'], 'traffic', a['roofline']['traffic'], 'ref', b['value'], 'ratio e2e', round(a['e2e']['value']/b['value'],1))"
