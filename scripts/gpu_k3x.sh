mkdir -p gpurun_out
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMLSORT_K3L_TIMING -I include"
for x in 0 1 2; do nvcc $F -DMLSORT_K3L_EXPT=$x -o /tmp/k3b$x scripts/k3_bench.cu; done
for x in 0 1 2; do echo "== expt $x"; /tmp/k3b$x | grep -E "best|phase"; done
