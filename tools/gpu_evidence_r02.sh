set -x
mkdir -p gpurun_out/r02ev
python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/r02ev/cfg2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cpqr_kernel -s 40 -c 1 -o gpurun_out/r02ev/cpqr_cfg2 python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/r02ev/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:core_fit -c 1 -o gpurun_out/r02ev/corefit_cfg2 python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/r02ev/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gauss -s 4 -c 1 -o gpurun_out/r02ev/gauss_cfg2 python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/r02ev/ncu3.log 2>&1
python tools/run_configs.py --cfg 3 --n 4096 --reps 1 --profile > gpurun_out/r02ev/cfg3_4096.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:core_fit -c 1 -o gpurun_out/r02ev/corefit_cfg3 python tools/run_configs.py --cfg 3 --n 4096 --reps 1 > gpurun_out/r02ev/ncu4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cpqr_kernel -s 30 -c 1 -o gpurun_out/r02ev/cpqr_cfg3 python tools/run_configs.py --cfg 3 --n 4096 --reps 1 > gpurun_out/r02ev/ncu5.log 2>&1
timeout 600 python tools/run_configs.py --cfg 3 --n 16384 --reps 1 --profile > gpurun_out/r02ev/cfg3_16384.log 2>&1
echo cfg3_16384 rc=$?
timeout 1200 python tools/run_configs.py --cfg 3 --n 65536 --reps 1 --profile > gpurun_out/r02ev/cfg3_65536.log 2>&1
echo cfg3_65536 rc=$?
tail -5 gpurun_out/r02ev/cfg3_65536.log
ls -la gpurun_out/r02ev
