timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
python tools/gemm_bench.py 16384 1664 832 > gpurun_out/gemm_t2.log 2>&1; echo rc=$?
for form in accumulate pairs; do
DMT_DCN_BWD=$form python bench.py --steps 30 --no-e2e --no-cpu > gpurun_out/bench_n1_$form.log 2>&1; echo rc=$?
done
