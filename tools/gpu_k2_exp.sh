# K2 experiment builds on the fixed dense config-2 product (tools/k2_bench.py); bits: 1 no MMA, 2 no eval, 4 no B copy, 8 no A writes
N=paper_2002_03400_b200/_native
for L in $N/libbfly_b200.so $N/libbfly_b200_*.so; do
  echo "== $(basename $L) $(BFLY_LIB=$PWD/$L python tools/k2_bench.py 2>&1 | tail -2 | head -1)"
done
