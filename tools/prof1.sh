set -x
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pooled_fwd -s 1 -c 1 -o gpurun_out/prof_lookup $CMD > gpurun_out/ncu2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 4 -c 2 -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bwd_update -s 1 -c 1 -o gpurun_out/prof_bwd $CMD > gpurun_out/ncu4.log 2>&1
echo rc=$?
ls -la gpurun_out
