# Smoke + GPU tests + bench on one B200 (no ncu): gpurun --timeout 900 -- bash tools/gpu_check.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/bench.log
