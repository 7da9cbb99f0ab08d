timeout 600 python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
for form in accumulate pairs; do
DMT_DCN_BWD=$form python bench.py --steps 30 --no-e2e --no-cpu > gpurun_out/bench_n1_$form.log 2>&1; echo rc=$?
done
DMT_DCN_BWD=pairs ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pairs.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1; echo rc=$?
