for k in 0 1 2 4 8; do DMT_TF32_KCHUNK=$k timeout 120 python tools/fp32_gemm_speed.py 2>&1 | grep -v Warn >> gpurun_out/g7_speed.log; done
timeout 900 python -m pytest tests/test_gpu_c2_parity.py tests/test_gpu_train.py -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/g7_tests.log 2>&1
echo "rc=$?" >> gpurun_out/g7_tests.log
