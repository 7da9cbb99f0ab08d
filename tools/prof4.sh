timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench12.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv $CMD > gpurun_out/ncu1.log 2>&1
echo rc=$?
