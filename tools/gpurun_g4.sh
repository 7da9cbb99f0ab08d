for v in none inline_side no_prepare both; do python tools/graph_debug3.py $v 2>&1 | grep -v Warn; done > gpurun_out/g4.log
