B="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu --no-e2e"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
P="python tools/profile_fill.py --config c2"
$P > gpurun_out/plain_prof.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_sobol_fast -s 1 -c 1 -o gpurun_out/prof_c2 $P > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
tail -3 gpurun_out/ncu_full.log
