timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $n --steps 30 --warmup 5 > gpurun_out/bench_n${n}.log 2>&1; echo bench_n${n}_rc=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 \
      tools/calibrate_costmodel.py --towers 2 --bench gpurun_out/bench_n4.log > gpurun_out/calib_n4.log 2>&1; echo calib_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 \
      bench.py --gpus 4 --towers 4 --steps 30 --warmup 5 --no-e2e > gpurun_out/bench_n4_t4.log 2>&1; echo bench_n4_t4_rc=$?
