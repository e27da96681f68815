# K2 trace-build experiment: full kernel vs no MMAs (mode 1) vs no evaluation (mode 2) vs neither (3)
mkdir -p gpurun_out/k2
for m in 0 1 2 3; do
  BFLY_OZ_MODE=$m BFLY_LIB=$PWD/paper_2002_03400_b200/_native/libbfly_b200_trace.so python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/k2/mode$m.log 2>&1
  echo "mode $m: $(grep '\[oz\] ctas 16384' gpurun_out/k2/mode$m.log | tail -1)"
done
