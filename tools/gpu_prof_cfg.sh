# ncu --set full of the search kernel on a cached config: CFG (cfg4), EFS (4000), DIST (warp-tree), OUT name
P="python bench.py --config ${CFG:-cfg4} --efs ${EFS:-4000} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --dist ${DIST:-warp-tree}"
$P > gpurun_out/prof_plain_${OUT:-cfg}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pag_search -s 2 -c 1 -o gpurun_out/prof_${OUT:-cfg} $P > gpurun_out/ncu_${OUT:-cfg}.log 2>&1; echo ncu=$?
tail -1 gpurun_out/prof_plain_${OUT:-cfg}.log | cut -c1-300
