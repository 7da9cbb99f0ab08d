timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 \
      bench.py --gpus 4 --steps 10 --warmup 3 --tables 100 --dim 256 --batch 4096 --no-e2e > gpurun_out/bench_n4_c4.log 2>&1; echo bench_n4_c4_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 \
      bench.py --gpus 2 --steps 20 --warmup 3 --pool-dist powerlaw > gpurun_out/bench_n2_pl.log 2>&1; echo bench_n2_pl_rc=$?
