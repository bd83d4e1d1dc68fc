# K3 DRAM bytes + bench (quick)
mkdir -p gpurun_out
NOTEST=1 bash scripts/gpu_quick.sh
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k3_local_sort -s 2 -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "dram__|gpu__time" 
