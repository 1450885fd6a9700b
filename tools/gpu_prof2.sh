B="python bench.py --steps 5 --warmup 3 --no-extra --no-cpu --no-e2e"
$B > gpurun_out/plain_bench2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_r01b.csv $B > gpurun_out/ncu_launch2.log 2>&1; echo launches rc=$?
for c in c2 c4 c3owen; do
  P="python tools/profile_fill.py --config $c"
  $P > gpurun_out/plain_$c.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_ -s 1 -c 1 -o gpurun_out/prof2_$c $P > gpurun_out/ncu2_$c.log 2>&1; echo $c rc=$?
done
R="python tools/profile_fill.py --config c5256"
$R > gpurun_out/plain_r2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render -s 1 -c 1 -o gpurun_out/prof2_c5 $R > gpurun_out/ncu2_c5.log 2>&1; echo c5 rc=$?
