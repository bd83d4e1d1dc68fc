# K1 keys-per-lane experiment: bench line with KGW = 8 (default) and 4
mkdir -p gpurun_out
for kg in 8 4; do
  MLSORT_NVCC_FLAGS="-DMLSORT_K1_KG=$kg" python -c "import paper_1805_04272_b200.build as b; b.build(force=True)" > /dev/null 2>&1
  echo "KG=$kg"; NOTEST=1 bash scripts/gpu_quick.sh
done
python -c "import paper_1805_04272_b200.build as b; b.build(force=True)" > /dev/null 2>&1
