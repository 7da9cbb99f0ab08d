timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_train.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
timeout 300 python tools/gemm_bench.py 16384 1664 832 > gpurun_out/gemm_t2.log 2>&1; echo rc=$?
timeout 300 python tools/gemm_bench.py 8192 3328 1664 > gpurun_out/gemm_t1.log 2>&1; echo rc=$?
timeout 300 python bench.py --steps 30 --no-e2e --no-cpu > gpurun_out/bench_n1.log 2>&1; echo rc=$?
