cd $GRAFT_REPO_ROOT
nproc > gpurun_out/g1_nproc.txt
timeout 900 python -m pytest tests/test_gpu_c2_parity.py tests/test_gpu_train.py -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/g1_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g1_tests.log
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g1_alltests.log 2>&1
echo "all rc=$?" >> gpurun_out/g1_alltests.log
