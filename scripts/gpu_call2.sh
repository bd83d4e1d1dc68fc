mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke2.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests2.log 2>&1; echo tests=$?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/k9 scripts/k9_pipes.cu && /tmp/k9 > gpurun_out/k9f.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_act2ILi9ELi8ELi2ELi2 -c 1 -o gpurun_out/k9act /tmp/k9 > gpurun_out/k9ncu.log 2>&1; echo ncu=$?
ls -la gpurun_out
