nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/k9 scripts/k9_pipes.cu && mkdir -p gpurun_out && /tmp/k9 > gpurun_out/k9e.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_act -o gpurun_out/k9act /tmp/k9 > gpurun_out/k9ncu.log 2>&1; echo ncu=$?
