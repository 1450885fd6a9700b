#!/bin/bash
# Round-2 evidence: the bench's launch list (cold-cache, serialised device
# times: compare shares) and full ncu captures of the hot kernels, each after
# its command ran clean without ncu. One GPU. Reports are summarised on the
# box (raw page CSV + tools/ncu_summary.py) and only the summaries come back.
#   bash tools/gpu_prof_r02.sh [launches] [config:kernel ...]
set -u
if [ "${1:-}" = "launches" ]; then
  shift
  B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
  $B > gpurun_out/plain_bench.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/r02_launches_bench.csv $B > gpurun_out/ncu_launches.log 2>&1
  echo launches rc=$?
fi
P="python tools/profile_fill.py"
for cfg in "$@"; do
  c=${cfg%%:*}; k=${cfg##*:}
  $P --config $c > gpurun_out/plain_$c.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o /tmp/r02_$c $P --config $c > gpurun_out/ncu_$c.log 2>&1
  echo $c rc=$?
  if [ -f /tmp/r02_$c.ncu-rep ]; then
    python tools/ncu_summary.py /tmp/r02_$c.ncu-rep > gpurun_out/r02_${c}_summary.txt 2>&1
    ncu -i /tmp/r02_$c.ncu-rep --page raw --csv > gpurun_out/r02_${c}_raw.csv 2>/dev/null
    python tools/ncu_hot.py /tmp/r02_$c.ncu-rep > gpurun_out/r02_${c}_hot.txt 2>&1 || true
  fi
done
