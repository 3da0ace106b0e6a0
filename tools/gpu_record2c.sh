# Round-2 record, part C: cfg-5 online inserts (20 reference insert batches, GPU refresh + search per phase)
R=gpurun_out/rec2c; mkdir -p $R
timeout 3000 python bench.py --config cfg5 --steps 10 --warmup 3 > $R/bench_cfg5.json 2> $R/bench_cfg5.err; echo cfg5=$?
tail -3 $R/bench_cfg5.err
