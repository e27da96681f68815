# A/B of the K2 slice schemes (6-slice default build vs the round-1 7-slice build), parity, cpqr captures
set -x
mkdir -p gpurun_out/ab
for rep in 1 2; do
  BFLY_LIB=$PWD/paper_2002_03400_b200/_native/libbfly_b200_oz7.so python tools/run_configs.py --cfg 2 4 --reps 4 --profile > gpurun_out/ab/oz7_$rep.log 2>&1
  python tools/run_configs.py --cfg 2 4 --reps 4 --profile > gpurun_out/ab/oz6_$rep.log 2>&1
done
python -m pytest tests/test_full_parity.py tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x -s > gpurun_out/ab/parity6.log 2>&1
echo parity6 rc=$?
python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/ab/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:matvec_oz -s 8 -c 1 -o gpurun_out/ab/oz6_k2 python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/ab/ncu_k2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cpqr_kernel -s 9 -c 1 -o gpurun_out/ab/cpqr_cfg2 python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/ab/ncu_cpqr2.log 2>&1
python tools/run_configs.py --cfg 3 --n 4096 --reps 1 > gpurun_out/ab/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cpqr_kernel -s 12 -c 1 -o gpurun_out/ab/cpqr_cfg3 python tools/run_configs.py --cfg 3 --n 4096 --reps 1 > gpurun_out/ab/ncu_cpqr3.log 2>&1
grep -h "construct" gpurun_out/ab/oz*_*.log
tail -3 gpurun_out/ab/parity6.log
