# Round-2 record, part B (cfg-3, cfg-4), on one B200. Outputs under gpurun_out/rec2b/.
R=gpurun_out/rec2b; mkdir -p $R
for c in cfg3 cfg4; do
  timeout 2400 python bench.py --config $c --steps 10 --warmup 3 > $R/bench_$c.json 2> $R/bench_$c.err; echo $c=$?
  E=$(python -c "import json; print(json.load(open('$R/bench_$c.json'))['config']['efS'])")
  N=$(python -c "import json; print(json.load(open('$R/bench_$c.json'))['config']['queries_per_step'])")
  echo "$c efS=$E nq=$N" > $R/op_$c.txt
  P="python bench.py --config $c --efs $E --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --print-units base -k regex:pag_search -s 3 -c 1 $P > $R/traffic_$c.csv 2> $R/traffic_$c.err; echo ncu_t$c=$?
  ncu --set full --clock-control none --import-source on -k regex:pag_search -s 3 -c 1 -o $R/full_$c $P > $R/ncu_full_$c.log 2>&1; echo ncu_f$c=$?
  python tools/ncu_summary.py $R/full_$c.ncu-rep 30 > $R/full_$c.txt 2>&1
done
timeout 900 python tools/gt_tc_bench.py cfg3 100 > $R/gt_cfg3.jsonl 2> $R/gt_cfg3.err; echo gt3=$?
timeout 900 python tools/gt_tc_bench.py cfg4 1000 > $R/gt_cfg4.jsonl 2> $R/gt_cfg4.err; echo gt4=$?
timeout 900 python tools/recall_curve.py cfg3 100 200 300 500 800 > $R/recall_qps_cfg3.json 2> $R/curve_cfg3.err; echo curve3=$?
# cfg-4 concurrency floor: one warp per SM (148 queries in flight; scratch + bitmaps ~67 MB, L2-resident)
PAG_GPU_WPB=1 PAG_GPU_MAX_BPS=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --print-units base -k regex:pag_search -s 3 -c 1 python bench.py --config cfg4 --efs 4000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $R/ncu_cfg4_wpb1_bps1.csv 2> $R/ncu_cfg4_wpb1_bps1.err; echo lowocc=$?
for f in $R/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('value'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"; done
