mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab/parity.log 2>&1; echo parity rc=$?; tail -2 gpurun_out/ab/parity.log
N=paper_2002_03400_b200/_native
for L in $N/libbfly_b200.so $N/libbfly_b200_*.so; do
  echo "== $(basename $L) $(BFLY_LIB=$PWD/$L python tools/k2_bench.py 2>&1 | tail -2 | head -1)"
done
bash tools/k2_ab.sh $N/libbfly_b200.so $(ls $N/libbfly_b200_*.so) 2>&1 | tee gpurun_out/ab/ab.txt
