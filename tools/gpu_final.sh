( time python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
( time python bench.py --impl reference ) > gpurun_out/bench_ref_default.json 2> gpurun_out/bench_ref_default.err; echo ref rc=$?
tail -3 gpurun_out/bench_default.err; tail -3 gpurun_out/bench_ref_default.err
