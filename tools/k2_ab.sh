# same-box A/B of two library builds on config 2: K2 ms per construction, alternating
A=${1:-paper_2002_03400_b200/_native/libbfly_b200.so}; Bl=${2}
for i in 1 2 3; do
  for L in $A $Bl; do
    echo "$L: $(BFLY_LIB=$PWD/$L python tools/run_configs.py --cfg 2 --reps 3 --profile 2>&1 | grep 'kernel kernel_matvec ' | awk '{print $6}') ms K2"
  done
done
