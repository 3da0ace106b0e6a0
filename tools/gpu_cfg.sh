# full-size bench of one config (builds/caches the index): CFG=cfg3 bash tools/gpu_cfg.sh
python bench.py --config ${CFG} --steps ${STEPS:-5} --warmup 3 ${EXTRA:-} > gpurun_out/b_${CFG}.json 2> gpurun_out/b_${CFG}.err; echo rc=$?
tail -12 gpurun_out/b_${CFG}.err
cat gpurun_out/b_${CFG}.json
