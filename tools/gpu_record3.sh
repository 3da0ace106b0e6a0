# Round-2 final record, part A (cfg-2 family + cfg-1 + construction), on one B200.
# Outputs under gpurun_out/rec3/. Every ncu pass runs only after the same
# command has exited 0 without ncu.
R=gpurun_out/rec3; mkdir -p $R
nvidia-smi > $R/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 400 --timeout-method=thread > $R/pytest_gpu.txt 2>&1; echo pytest=$?
tail -2 $R/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.txt 2>&1; echo smoke=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $R/bench_ref.json 2> $R/bench_ref.err; echo ref=$?
timeout 900 python bench.py --steps 20 --warmup 5 > $R/bench_cfg2.json 2> $R/bench_cfg2.err; echo cfg2=$?
timeout 900 python bench.py --steps 20 --warmup 5 --dist exact > $R/bench_cfg2_exact.json 2> $R/bench_cfg2_exact.err; echo cfg2x=$?
for d in 0,0 0,0,0,0; do timeout 900 python bench.py --shard abi --devices $d --steps 8 --warmup 4 > $R/bench_abi_$d.json 2> $R/bench_abi_$d.err; echo abi$d=$?; done
timeout 900 python bench.py --config cfg1 --steps 20 --warmup 5 > $R/bench_cfg1.json 2> $R/bench_cfg1.err; echo cfg1=$?
timeout 900 python bench.py --mode construction --steps 5 --warmup 3 > $R/bench_cons.json 2> $R/bench_cons.err; echo cons=$?
timeout 900 python tools/gt_tc_bench.py cfg2 10 100 1000 > $R/gt_cfg2.jsonl 2> $R/gt_cfg2.err; echo gt=$?
timeout 900 python tools/gt_tc_bench.py cfg2 10 --lists > $R/gt_cfg2_lists.jsonl 2> $R/gt_cfg2_lists.err; echo gtl=$?
timeout 900 python tools/recall_curve.py cfg2 10 20 40 60 70 80 100 150 200 300 400 > $R/recall_qps_cfg2.json 2> $R/curve_cfg2.err; echo curve=$?
# ncu: launch list of the default bench command (timed steps), DRAM bytes per launch, one full capture per mode
P="python bench.py --efs 70 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --print-units base --log-file $R/launches_cfg2.csv $P > $R/ncu_launches.log 2>&1; echo ncu_l=$?
for d in warp-tree exact; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --print-units base -k regex:pag_search -s 3 -c 1 $P --dist $d > $R/traffic_cfg2_$d.csv 2> $R/traffic_cfg2_$d.err; echo ncu_t$d=$?
  ncu --set full --clock-control none --import-source on -k regex:pag_search -s 3 -c 1 -o /tmp/full_cfg2_$d $P --dist $d > $R/ncu_full_cfg2_$d.log 2>&1; echo ncu_f$d=$?
  python tools/ncu_summary.py /tmp/full_cfg2_$d.ncu-rep 30 > $R/full_cfg2_$d.txt 2>&1
done
C="python bench.py --mode construction --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --print-units base -k regex:pag_search -s 3 -c 1 $C > $R/traffic_cons.csv 2> $R/traffic_cons.err; echo ncu_tc=$?
ncu --set full --clock-control none --import-source on -k regex:pag_search -s 3 -c 1 -o /tmp/full_cons $C > $R/ncu_full_cons.log 2>&1; echo ncu_fc=$?
python tools/ncu_summary.py /tmp/full_cons.ncu-rep 30 > $R/full_cons.txt 2>&1
G="python tools/gt_tc_bench.py cfg2 1000"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__inst_executed_pipe_uma.sum --clock-control none --csv --print-units base -k regex:gt_tc -c 12 $G > $R/ncu_gt_cfg2.csv 2> $R/ncu_gt_cfg2.err; echo ncu_gt=$?
for f in $R/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('value'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"; done
R=gpurun_out/rec3; mkdir -p $R
for c in cfg3 cfg4; do
  timeout 2400 python bench.py --config $c --steps 10 --warmup 3 > $R/bench_$c.json 2> $R/bench_$c.err; echo $c=$?
  E=$(python -c "import json; print(json.load(open('$R/bench_$c.json'))['config']['efS'])")
  N=$(python -c "import json; print(json.load(open('$R/bench_$c.json'))['config']['queries_per_step'])")
  echo "$c efS=$E nq=$N" > $R/op_$c.txt
  P="python bench.py --config $c --efs $E --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --print-units base -k regex:pag_search -s 3 -c 1 $P > $R/traffic_$c.csv 2> $R/traffic_$c.err; echo ncu_t$c=$?
  ncu --set full --clock-control none --import-source on -k regex:pag_search -s 3 -c 1 -o /tmp/full_$c $P > $R/ncu_full_$c.log 2>&1; echo ncu_f$c=$?
  python tools/ncu_summary.py /tmp/full_$c.ncu-rep 30 > $R/full_$c.txt 2>&1
done
timeout 900 python tools/gt_tc_bench.py cfg3 100 > $R/gt_cfg3.jsonl 2> $R/gt_cfg3.err; echo gt3=$?
timeout 900 python tools/gt_tc_bench.py cfg4 1000 > $R/gt_cfg4.jsonl 2> $R/gt_cfg4.err; echo gt4=$?
timeout 900 python tools/recall_curve.py cfg3 100 200 300 500 800 > $R/recall_qps_cfg3.json 2> $R/curve_cfg3.err; echo curve3=$?
for f in $R/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('value'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"; done
timeout 3000 python bench.py --config cfg5 --steps 10 --warmup 3 > $R/bench_cfg5.json 2> $R/bench_cfg5.err; echo cfg5=$?
for m in fast exact; do timeout 300 python tools/phases.py cfg2 70 $m > $R/phases_cfg2_$m.txt 2>&1; timeout 600 python tools/phases.py cfg3 100 $m > $R/phases_cfg3_$m.txt 2>&1; done
