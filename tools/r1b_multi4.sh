timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 \
      tools/calibrate_costmodel.py --towers 2 --bench gpurun_out/bench_n4.log > gpurun_out/calib_n4.log 2>&1; echo calib_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 \
      bench.py --gpus 4 --steps 30 --warmup 5 --top dcn --no-e2e > gpurun_out/bench_n4_top.log 2>&1; echo bench_n4_top_rc=$?
timeout 600 python bench.py --steps 30 --top dcn --no-cpu > gpurun_out/bench_n1_top.log 2>&1; echo bench_n1_top_rc=$?
