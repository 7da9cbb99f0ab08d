timeout 300 python tools/graph_debug5.py fwd 2>&1 | grep -v Warn > gpurun_out/g6.log
timeout 300 python tools/graph_debug5.py step 2>&1 | grep -v Warn >> gpurun_out/g6.log
