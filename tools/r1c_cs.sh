timeout 120 python tools/colsum_bench.py > gpurun_out/cs_bench.log 2>&1; echo rc=$?
