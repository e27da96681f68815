mkdir -p gpurun_out/b3
timeout 900 python -m pytest tests/test_full_parity.py tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x > gpurun_out/b3/parity.log 2>&1; echo parity rc=$?; tail -2 gpurun_out/b3/parity.log
python tools/apply_bench.py --synth --ks 1,2,4,8,16,32,66 --reps 20 > gpurun_out/b3/apply4.log 2>&1; cat gpurun_out/b3/apply4.log | tail -7
python tools/apply_bench.py --synth --ks 16 --reps 3 > /dev/null 2>&1 && \
BFLY_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b3/apply4_k16_launches.csv python tools/apply_bench.py --synth --ks 16 --reps 3 > /dev/null 2>&1
BFLY_NO_GRAPHS=1 ncu --set full --clock-control none --import-source on -k regex:bgemm -s 40 -c 3 -o gpurun_out/b3/apply4_k16 python tools/apply_bench.py --synth --ks 16 --reps 3 > gpurun_out/b3/ncu_apply.log 2>&1
python tools/run_configs.py --cfg 2 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:cpqr_kernel -s 8 -c 1 -o gpurun_out/b3/cpqr_cfg2 python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/b3/ncu_cpqr.log 2>&1
echo done
