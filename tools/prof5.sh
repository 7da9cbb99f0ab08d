timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; tail -1 gpurun_out/pytest.log
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench13.log 2>&1
CMD="python tools/gemm_bench.py"
$CMD > gpurun_out/gemm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 23 -c 1 -o gpurun_out/prof_dcnbwd $CMD > gpurun_out/ncu5.log 2>&1
echo rc=$?
