timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
timeout 600 python bench.py --steps 30 --no-cpu > gpurun_out/bench_n1.log 2>&1; echo bench_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_n2.log 2>&1; echo bench_n2_rc=$?
