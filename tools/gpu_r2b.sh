mkdir -p gpurun_out/r2b
timeout 1200 python -m pytest tests -x -q -m gpu --timeout 400 --timeout-method=thread > gpurun_out/r2b/pytest_gpu.txt 2>&1; echo pytest=$?
tail -5 gpurun_out/r2b/pytest_gpu.txt
grep -E "id sets differ" gpurun_out/r2b/pytest_gpu.txt | head
timeout 900 python tools/gt_tc_bench.py cfg2 10 100 1000 > gpurun_out/r2b/gt_cfg2.jsonl 2> gpurun_out/r2b/gt_cfg2.err; echo gt=$?
cat gpurun_out/r2b/gt_cfg2.jsonl
