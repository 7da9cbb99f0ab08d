timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=5 > gpurun_out/g8_tests.log 2>&1
echo "rc=$?" >> gpurun_out/g8_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g8_bench.json 2> gpurun_out/g8_bench.err
echo "bench rc=$?" >> gpurun_out/g8_bench.err
