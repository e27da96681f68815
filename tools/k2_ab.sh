# same-box A/B of library builds on config 2: K2 ms per construction, alternating
# usage: tools/k2_ab.sh lib1.so lib2.so [lib3.so ...]
for i in 1 2 3; do
  for L in "$@"; do
    echo "$(basename $L): $(BFLY_LIB=$PWD/$L python tools/run_configs.py --cfg 2 --reps 3 --profile 2>&1 | grep 'kernel kernel_matvec ' | awk '{print $6}') ms K2"
  done
done
