# Round-end evidence: default bench (ours + reference arm), the ncu launch
# list of the headline command, and one ncu --set full capture per hot kernel
# (each capture only after the same command exited 0 without ncu).
#   bash tools/gpu_prof_final.sh bench        # benches + launch list
#   bash tools/gpu_prof_final.sh c2 c4 ...    # captures (<= 4 per call: 64 MiB)
for what in "$@"; do
  if [ "$what" = bench ]; then
    python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
    python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo ref rc=$?
    B="python bench.py --steps 5 --warmup 3 --no-extra --no-cpu --no-e2e"
    $B > gpurun_out/plain_headline.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $B > gpurun_out/ncu_launch_final.log 2>&1; echo launches rc=$?
  else
    P="python tools/profile_fill.py --config $what"
    $P > gpurun_out/plain_$what.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 1 -c 1 -o gpurun_out/final_$what $P > gpurun_out/ncu_final_$what.log 2>&1; echo $what rc=$?
  fi
done
