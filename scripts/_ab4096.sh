for v in default lib_biggen lib_big3; do
  if [ $v = default ]; then unset QSDP_LIB_PATH; else export QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/$v.so; fi
  echo "=== $v"; python scripts/prof_kernels.py --bucket 4096 --gbits 4 --reps 11 | grep -E "K1|K2"
done
