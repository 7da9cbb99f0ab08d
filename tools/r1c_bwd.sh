for v in 1 10 11 12 13; do echo "variant $v"; DMT_BWD_VARIANT=$v timeout 120 python tools/lookup_bench.py bf16 2>&1 | tail -1; done > gpurun_out/bwd_variants.log 2>&1
for v in 10 11 12 13; do echo "variant $v"; DMT_BWD_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_train.py -x -q -k "embedding_backward" 2>&1 | tail -2; done > gpurun_out/bwd_variant_tests.log 2>&1
echo done
