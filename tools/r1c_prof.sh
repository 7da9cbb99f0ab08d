# r1c evidence: N=1 launch list + ncu --set full of the embedding-backward apply (new default), then N=2 / N=4 benches
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
(export CUDA_VISIBLE_DEVICES=0
 $CMD > gpurun_out/plain_c.log 2>&1 && \
 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv $CMD > gpurun_out/ncu_c_l.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:bwd_update -s 1 -c 1 -o gpurun_out/r1c_bwd_update $CMD > gpurun_out/ncu_c_a.log 2>&1
 echo prof_rc=$?)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.log 2>&1; echo bench_n2_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
      bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.log 2>&1; echo bench_n4_rc=$?
