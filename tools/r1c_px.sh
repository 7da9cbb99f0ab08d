timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_exchange.py -x -q > gpurun_out/multi_tests.log 2>&1; echo tests_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
      bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.log 2>&1; echo bench_n4_rc=$?
