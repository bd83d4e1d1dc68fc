# A/B of a compile-time macro on one box: usage bash scripts/gpu_ab.sh "-DX=0" "-DX=1"
mkdir -p gpurun_out
for fl in "$1" "$2" "$1" "$2"; do
  MLSORT_NVCC_FLAGS="$fl" python -c "import paper_1805_04272_b200.build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== $fl"; NOTEST=1 bash scripts/gpu_quick.sh
done
python -c "import paper_1805_04272_b200.build as b; b.build(force=True)" > /dev/null 2>&1
