# r1 evidence: launch list of one bench step + full captures of the top kernels
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pooled_fwd -s 2 -c 1 -o gpurun_out/r1_lookup_fwd $CMD > gpurun_out/ncu_a.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bwd_update -s 2 -c 1 -o gpurun_out/r1_bwd_update $CMD > gpurun_out/ncu_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 16 -c 4 -o gpurun_out/r1_gemms $CMD > gpurun_out/ncu_c.log 2>&1
echo rc=$?
