# re-entry check: GPU parity tests + N=1 bench + smoke
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/bench_n1.log 2>&1; echo bench_rc=$?
