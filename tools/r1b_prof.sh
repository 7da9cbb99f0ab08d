timeout 600 python -m pytest tests/test_gpu_train.py -q -k "bce" > gpurun_out/gpu_tests_bce.log 2>&1; echo tests_rc=$?
bash tools/prof8.sh
python tools/ncu_summary.py gpurun_out/r1b_lookup_fwd.ncu-rep "pooled lookup fwd, C2 bf16 26x1Mx128 B=8192 L=20 (bench.py step), r1b" --json gpurun_out/r1b_lookup_fwd.json > gpurun_out/r1b_ncu_lookup_fwd.txt
python tools/ncu_summary.py gpurun_out/r1b_gemms.ncu-rep "all 12 DCN TM GEMM launches of one bench step (tcgen05), C2 bf16 N=1, r1b" --json gpurun_out/r1b_gemms.json > gpurun_out/r1b_ncu_gemms.txt
rm -f gpurun_out/r1b_gemms.ncu-rep
ls -la gpurun_out/
