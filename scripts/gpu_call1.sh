set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/k9 scripts/k9_pipes.cu && timeout 120 /tmp/k9 > gpurun_out/k9.txt 2>&1; echo k9=$?
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
