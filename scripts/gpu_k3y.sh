mkdir -p gpurun_out
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMLSORT_K3L_TIMING -I include"
nvcc $F -o /tmp/k3b scripts/k3_bench.cu
echo "== fb14 NT1024"; /tmp/k3b | grep -E "best|phase"
echo "== fb13 NT1024"; K3_FB13=1 /tmp/k3b | grep -E "best|phase"
echo "== fb13 NT512 x2"; K3_FB13=1 K3_NT512=1 /tmp/k3b | grep -E "best|phase|mid"
