CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; tail -2 gpurun_out/pytest.log
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bwd_update_fast -s 1 -c 1 -o gpurun_out/prof_bwd3 $CMD > gpurun_out/ncu4.log 2>&1
echo rc=$?
