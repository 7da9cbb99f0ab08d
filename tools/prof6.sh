CMD="python tools/gemm_bench.py"
$CMD > gpurun_out/gemm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 115 -c 1 -o gpurun_out/prof_dcnbwd $CMD > gpurun_out/ncu5.log 2>&1
echo rc=$?
