# DRAM bytes per search launch (ncu) on the final sources, every recorded config, then the
# default bench line again. Outputs under gpurun_out/fin/.
R=gpurun_out/fin; mkdir -p $R
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --print-units base -k regex:pag_search -s 3 -c 1"
timeout 900 python bench.py --steps 10 --warmup 3 > $R/bench_cfg2.json 2> $R/bench_cfg2.err; echo cfg2=$?
for d in warp-tree exact; do ncu $M python bench.py --efs 70 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --dist $d > $R/traffic_cfg2_$d.csv 2> $R/t2$d.err; echo t2$d=$?; done
ncu $M python bench.py --mode construction --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $R/traffic_cons.csv 2> $R/tc.err; echo tc=$?
timeout 1500 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $R/bench_cfg3_quick.json 2> $R/b3.err; echo b3=$?
ncu $M python bench.py --config cfg3 --efs 100 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $R/traffic_cfg3.csv 2> $R/t3.err; echo t3=$?
timeout 2400 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $R/bench_cfg4_quick.json 2> $R/b4.err; echo b4=$?
ncu $M python bench.py --config cfg4 --efs 4000 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $R/traffic_cfg4.csv 2> $R/t4.err; echo t4=$?
for f in $R/bench_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['roofline']['source_sha'], d['config']['efS'])"; done
