# K2 change check: timings of configs 2 / 1 / 0 (+ kernel table) and the GPU parity suites
mkdir -p gpurun_out/k2
tag=${1:-cur}
python tools/run_configs.py --cfg 2 1 0 --reps 4 --profile > gpurun_out/k2/$tag.log 2>&1; echo timing rc=$?
grep -h "rep \|kernel_matvec \|cfg " gpurun_out/k2/$tag.log | head -30
if [ "${2:-parity}" = "parity" ]; then
  timeout 900 python -m pytest tests/test_full_parity.py tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x > gpurun_out/k2/parity_$tag.log 2>&1; echo parity rc=$?
  tail -3 gpurun_out/k2/parity_$tag.log
fi
