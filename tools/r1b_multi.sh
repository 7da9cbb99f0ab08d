# multi-GPU check: NCCL/peer parity tests + bench at N=2,4 (peer and nccl fabrics)
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_tests.log 2>&1; echo tests_rc=$?
for n in 2 4; do
  for fab in peer nccl; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $n --steps 30 --warmup 5 --no-e2e --fabric $fab > gpurun_out/bench_n${n}_${fab}.log 2>&1; echo bench_n${n}_${fab}_rc=$?
  done
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
      bench.py --gpus 4 --towers 4 --steps 30 --warmup 5 --no-e2e > gpurun_out/bench_n4_t4.log 2>&1; echo bench_n4_t4_rc=$?
