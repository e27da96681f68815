# structured butterfly black box: parity with the padded products, config-4 timings
set -x
mkdir -p gpurun_out/st
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "structured or synthetic_exact or config_parity or virtual_ranks" -p no:cacheprovider > gpurun_out/st/tests.log 2>&1; echo tests rc=$?; tail -15 gpurun_out/st/tests.log
python tools/run_configs.py --cfg 4 --reps 3 --profile > gpurun_out/st/cfg4.txt 2>&1; echo rc=$?
BFLY_NO_STRUCT_APPLY=1 python tools/run_configs.py --cfg 4 --reps 3 > gpurun_out/st/cfg4_padded.txt 2>&1
python tools/run_configs.py --cfg 4 --reps 3 --c64 > gpurun_out/st/cfg4_c64.txt 2>&1
grep -h "cfg 4\|rep \|transfer\|leaf" gpurun_out/st/cfg4.txt | head -40
grep -h "cfg 4" gpurun_out/st/cfg4_padded.txt gpurun_out/st/cfg4_c64.txt
