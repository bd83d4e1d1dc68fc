# K3 v7 check: standalone phase timing, GPU parity, C2 bench line
mkdir -p gpurun_out
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMLSORT_K3L_TIMING -I include"
nvcc $F -o /tmp/k3b scripts/k3_bench.cu
echo "== k3 bench"; /tmp/k3b
echo "== k3 bench verify"; K3_VERIFY=1 /tmp/k3b
echo "== k3 bench NT512"; K3_NT512=1 /tmp/k3b
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --steps 10 --warmup 3 2>&1 | tail -1
