# A/B of experiment builds: bash scripts/_ab.sh VARIANT... (r1 = the round-1 tree copy; default = in-tree lib)
R1=paper_2302_02390_b200/_variants/r1
for rep in 1 2; do
for v in "$@"; do
  echo "=== $v"
  if [ $v = r1 ]; then python $R1/scripts/prof_kernels.py --reps 11 | grep -E "K1|K2"; python $R1/scripts/prof_fused.py --reps 4 | tail -2;
  else
    if [ $v = default ]; then unset QSDP_LIB_PATH; else export QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/$v.so; fi
    python scripts/prof_kernels.py --reps 11 | grep -E "K1|K2"; python scripts/prof_fused.py --reps 4 | tail -2
    unset QSDP_LIB_PATH
  fi
done; done
