python tools/gemm_bench.py 16384 1664 832 > gpurun_out/gemm_t2.log 2>&1; echo rc=$?
python tools/gemm_bench.py 8192 3328 1664 > gpurun_out/gemm_t1.log 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/gemm_t2_cross python tools/gemm_bench.py 16384 1664 832 > gpurun_out/ncu_g.log 2>&1; echo rc=$?
