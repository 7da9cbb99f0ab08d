# r1b evidence: N=1 launch list + ncu --set full of the lookup and of one step's GEMMs (traffic.json source)
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain8.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv $CMD > gpurun_out/ncu8_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pooled_fwd -s 1 -c 1 -o gpurun_out/r1b_lookup_fwd $CMD > gpurun_out/ncu8_a.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 12 -c 12 -o gpurun_out/r1b_gemms $CMD > gpurun_out/ncu8_b.log 2>&1
echo rc=$?
