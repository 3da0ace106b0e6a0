# Round record on one B200: parity tests, the default bench line (cfg2), the
# reference arm, cfg3 / cfg4 / construction bench lines, the ncu launch list
# of the cfg2 bench command, one --set full capture of the search kernel,
# QPS-recall curves (cfg2, cfg3) and, with WITH_CFG5=1, the online-insert run.
# Outputs under gpurun_out/rec/.
mkdir -p gpurun_out/rec
timeout 600 python -m pytest tests -x -q -m gpu --timeout 200 --timeout-method=thread > gpurun_out/rec/pytest_gpu.txt 2>&1; echo pytest=$?
tail -2 gpurun_out/rec/pytest_gpu.txt
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/rec/bench_ref.json 2> gpurun_out/rec/bench_ref.err; echo ref=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/rec/bench_cfg2.json 2> gpurun_out/rec/bench_cfg2.err; echo cfg2=$?
python bench.py --config cfg3 --steps 10 --warmup 3 > gpurun_out/rec/bench_cfg3.json 2> gpurun_out/rec/bench_cfg3.err; echo cfg3=$?
python bench.py --config cfg4 --steps 5 --warmup 3 > gpurun_out/rec/bench_cfg4.json 2> gpurun_out/rec/bench_cfg4.err; echo cfg4=$?
python bench.py --mode construction --steps 5 --warmup 3 > gpurun_out/rec/bench_cons.json 2> gpurun_out/rec/bench_cons.err; echo cons=$?
python bench.py --config cfg1 --steps 20 --warmup 5 > gpurun_out/rec/bench_cfg1.json 2> gpurun_out/rec/bench_cfg1.err; echo cfg1=$?
P="python bench.py --efs 70 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rec/launches_cfg2.csv $P > gpurun_out/rec/ncu1.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:pag_search -s 2 -c 1 -o gpurun_out/rec/prof_cfg2 $P > gpurun_out/rec/ncu2.log 2>&1; echo ncu2=$?
timeout 900 python tools/recall_curve.py cfg2 10 20 40 60 70 80 100 150 200 300 400 600 > gpurun_out/rec/recall_qps_cfg2.json 2> gpurun_out/rec/curve_cfg2.err; echo curve2=$?
timeout 900 python tools/recall_curve.py cfg3 100 200 300 500 800 > gpurun_out/rec/recall_qps_cfg3.json 2> gpurun_out/rec/curve_cfg3.err; echo curve3=$?
if [ -n "$WITH_CFG5" ]; then timeout 1700 python bench.py --config cfg5 --steps 10 --warmup 3 > gpurun_out/rec/bench_cfg5.json 2> gpurun_out/rec/bench_cfg5.err; echo cfg5=$?; fi
for f in gpurun_out/rec/bench_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d.get('value'), d.get('roofline',{}).get('frac'), d.get('e2e',{}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"; done
