# Halton fill: parity subset, timings, one ncu --set full capture of k_halton_tiled.
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "radical or halton" -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/exp_halton.py
P="python tools/profile_fill.py --config halton"
$P > gpurun_out/plain_halton.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_halton -s 1 -c 1 -o gpurun_out/prof_halton $P > gpurun_out/ncu_halton.log 2>&1; echo halton rc=$?
