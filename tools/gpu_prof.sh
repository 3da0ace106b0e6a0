# ncu capture of the search kernel on the cached cfg2 index (run after a bench on the same box)
P="python bench.py --efs ${EFS:-70} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --dist ${DIST:-warp-tree}"
$P > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:pag_search -s 2 -c 1 -o gpurun_out/prof_search $P > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
tail -2 gpurun_out/prof_plain.log
