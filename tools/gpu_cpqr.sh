# CPQR for blocks of 33..64 rows: register-resident kernel (default) against the shared-memory forms
# (BFLY_CPQR_NH=2: four warps, two lanes per column; =1: two warps, lane per column): parity + config-4 / config-1 timing
set -x
mkdir -p gpurun_out/cq
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_full_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/cq/tests.log 2>&1; echo tests rc=$?; tail -4 gpurun_out/cq/tests.log
python tools/run_configs.py --cfg 4 1 --reps 4 --profile > gpurun_out/cq/reg.txt 2>&1
BFLY_CPQR_NH=2 python tools/run_configs.py --cfg 4 1 --reps 4 --profile > gpurun_out/cq/nh2.txt 2>&1
BFLY_CPQR_NH=1 python tools/run_configs.py --cfg 4 1 --reps 4 --profile > gpurun_out/cq/nh1.txt 2>&1
python tools/run_configs.py --cfg 4 --reps 3 --c64 --profile > gpurun_out/cq/reg_c64.txt 2>&1
grep -h "^cfg\|kernel cpqr" gpurun_out/cq/reg.txt gpurun_out/cq/nh2.txt gpurun_out/cq/nh1.txt gpurun_out/cq/reg_c64.txt
