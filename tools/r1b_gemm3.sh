timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k gemm > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
python tools/gemm_bench.py 16384 1664 832 > gpurun_out/gemm_t2.log 2>&1; echo rc=$?
python tools/gemm_bench.py 8192 3328 1664 > gpurun_out/gemm_t1.log 2>&1; echo rc=$?
