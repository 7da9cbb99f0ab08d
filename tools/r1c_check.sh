timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
timeout 600 python bench.py > gpurun_out/bench_n1.log 2>&1; echo bench_rc=$?
timeout 120 python tools/lookup_bench.py bf16 > gpurun_out/lookup_bench.log 2>&1; echo rc=$?
