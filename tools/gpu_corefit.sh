# K6 core fit with the Jacobi operands in shared memory (BFLY_COREFIT_SMEM=0: global scratch, the previous form)
set -x
mkdir -p gpurun_out/cf
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_full_parity.py tests/test_acceptance_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/cf/tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/cf/tests.log
python tools/run_configs.py --cfg 0 1 2 4 --reps 4 --profile > gpurun_out/cf/smem.txt 2>&1
BFLY_COREFIT_SMEM=0 python tools/run_configs.py --cfg 0 1 2 4 --reps 4 --profile > gpurun_out/cf/glob.txt 2>&1
python tools/run_configs.py --cfg 3 --n 4096 --reps 3 --profile > gpurun_out/cf/cfg3_smem.txt 2>&1
BFLY_COREFIT_SMEM=0 python tools/run_configs.py --cfg 3 --n 4096 --reps 3 --profile > gpurun_out/cf/cfg3_glob.txt 2>&1
echo "== shared"; grep -h "^cfg\|kernel core_fit" gpurun_out/cf/smem.txt gpurun_out/cf/cfg3_smem.txt
echo "== global"; grep -h "^cfg\|kernel core_fit" gpurun_out/cf/glob.txt gpurun_out/cf/cfg3_glob.txt
