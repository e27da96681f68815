# config-4 apply at k = 8 / 16 / 32 under the stage-kernel knobs
for cfg in "" "BFLY_STAGE_WPE=4" "BFLY_STAGE_WPE=8" "BFLY_NO_STAGE_GEMM=1"; do
  echo "== $cfg"
  env $cfg python tools/apply_bench.py --synth --ks 8,16,32 --reps 20 2>&1 | tail -3
done
