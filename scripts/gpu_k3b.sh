mkdir -p gpurun_out
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMLSORT_K3L_TIMING -I include"
nvcc $F -o /tmp/k3b scripts/k3_bench.cu
sed 's/        constexpr bool kCacheKeys = sizeof(KeyT) == 4 \&\& !PERM;/        constexpr bool kCacheKeys = false;/' paper_1805_04272_b200/csrc/k3_local.cuh > /tmp/k3_local_nokeys.cuh
sed 's#../paper_1805_04272_b200/csrc/k3_local.cuh#/tmp/k3_local_nokeys.cuh#' scripts/k3_bench.cu > /tmp/k3_bench_nokeys.cu
cp paper_1805_04272_b200/csrc/common.cuh paper_1805_04272_b200/csrc/k3_sort.cuh /tmp/
nvcc $F -o /tmp/k3b_nk /tmp/k3_bench_nokeys.cu
for v in "" 1; do
  echo "== keys cached, verify=$v"; env ${v:+K3_VERIFY=1} /tmp/k3b
  echo "== fine only, verify=$v"; env ${v:+K3_VERIFY=1} /tmp/k3b_nk
done
