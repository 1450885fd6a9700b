#!/bin/bash
# Round-2 evidence: the bench's launch list (cold-cache, serialised device
# times: compare shares) and full ncu captures of the hot kernels, each after
# its command ran clean without ncu. One GPU.
set -u
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain_bench.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r02_launches_bench.csv $B > gpurun_out/ncu_launches.log 2>&1
echo launches rc=$?
P="python tools/profile_fill.py"
for cfg in "c2:k_sobol_fast" "halton:k_tma" "c64:k_render" "c5iph:k_render" "bench-pixel-shifted-lattice:k_bench" "bench-halton-tabled:k_bench" "c4:k_lattice_fast" "c3owen:k_sobol_fast"; do
  c=${cfg%%:*}; k=${cfg##*:}
  $P --config $c > gpurun_out/plain_$c.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/r02_$c $P --config $c > gpurun_out/ncu_$c.log 2>&1
  echo $c rc=$?
done
