timeout 300 python tools/graph_debug4.py 2>&1 | grep -v Warn > gpurun_out/g5.log
for k in 0 1 2 4 8; do DMT_TF32_KCHUNK=$k timeout 120 python tools/fp32_accuracy.py > gpurun_out/g5_acc$k.log 2>&1; done
