DMT_BENCH_VERBOSE=1 timeout 600 python -X faulthandler bench.py --steps 10 --warmup 3 > gpurun_out/g9_bench.json 2> gpurun_out/g9_bench.err
echo "bench rc=$?" >> gpurun_out/g9_bench.err
