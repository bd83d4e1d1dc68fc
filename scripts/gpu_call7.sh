mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke7.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests7.log 2>&1; echo tests=$?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo bench=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o /tmp/k1b scripts/k1_bench.cu 2>/dev/null && /tmp/k1b > gpurun_out/k1b_2.txt 2>&1
