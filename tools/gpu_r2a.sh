# round-2 check: GPU tests, default bench line, reference arm, ABI-sharded bench on 2 replicas
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 --timeout-method=thread > gpurun_out/r2a/pytest_gpu.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/r2a/pytest_gpu.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2a/bench_ref.json 2> gpurun_out/r2a/bench_ref.err; echo ref=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a/bench_cfg2.json 2> gpurun_out/r2a/bench_cfg2.err; echo cfg2=$?
timeout 600 python bench.py --shard abi --devices 0,0 --steps 8 --warmup 4 > gpurun_out/r2a/bench_abi2.json 2> gpurun_out/r2a/bench_abi2.err; echo abi=$?
tail -3 gpurun_out/r2a/bench_cfg2.err
