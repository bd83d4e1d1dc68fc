mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build3.log 2>&1; echo build=$?
timeout 600 python -m pytest tests -x -q -m gpu -k "test_sort_sizes or full_config_exact" > gpurun_out/gputests3.log 2>&1; echo tests=$?
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/b3_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_predict -s 1 -c 1 -o gpurun_out/k1v2 $B > gpurun_out/ncu_k1.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k3_local -s 1 -c 1 -o gpurun_out/k3v2 $B > gpurun_out/ncu_k3.log 2>&1; echo ncu3=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/k9 scripts/k9_pipes.cu && /tmp/k9 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_act2<9, 4, 4" -c 1 -o gpurun_out/k9act /tmp/k9 > gpurun_out/k9ncu.log 2>&1; echo ncu9=$?
ls -la gpurun_out
