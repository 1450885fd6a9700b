set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; nproc; free -g | head -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke1.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -q -rA --timeout 600 -p no:cacheprovider > gpurun_out/gputests1.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/gputests1.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
