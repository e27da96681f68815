# basis projection answered by the butterfly black box (BFLY_NO_LEAF_FUSE=1: plain structured products + the factorizer's chain)
set -x
mkdir -p gpurun_out/fu
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/fu/tests.log 2>&1; echo tests rc=$?; tail -4 gpurun_out/fu/tests.log
python tools/run_configs.py --cfg 4 --reps 6 --profile > gpurun_out/fu/fused.txt 2>&1
BFLY_NO_LEAF_FUSE=1 python tools/run_configs.py --cfg 4 --reps 4 --profile > gpurun_out/fu/plain.txt 2>&1
python tools/run_configs.py --cfg 4 --reps 6 --c64 --profile > gpurun_out/fu/fused_c64.txt 2>&1
echo "== fused"; grep -h "rep \|^cfg\|kernel " gpurun_out/fu/fused.txt | cut -c1-170
echo "== fused c64"; grep -h "rep \|^cfg\|kernel " gpurun_out/fu/fused_c64.txt | cut -c1-170
echo "== separate"; grep -h "^cfg" gpurun_out/fu/plain.txt | cut -c1-170
