# round-2 ncu evidence: K2 transfer-level launch, config-4 k=16 apply stage, bench launch list
mkdir -p gpurun_out/ev2
python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/ev2/plain_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:matvec_oz -s 8 -c 1 -o gpurun_out/ev2/k2_cfg2 python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/ev2/ncu_k2.log 2>&1
python tools/apply_bench.py --synth --ks 16 --reps 3 > gpurun_out/ev2/plain_apply.log 2>&1 && \
BFLY_NO_GRAPHS=1 ncu --set full --clock-control none --import-source on -k regex:bgemm_stage -s 40 -c 2 -o gpurun_out/ev2/apply4_k16 python tools/apply_bench.py --synth --ks 16 --reps 3 > gpurun_out/ev2/ncu_apply.log 2>&1
python tools/apply_bench.py --synth --ks 1 --reps 3 > gpurun_out/ev2/plain_apply1.log 2>&1 && \
BFLY_NO_GRAPHS=1 ncu --set full --clock-control none --import-source on -k regex:bgemm_stage -s 40 -c 2 -o gpurun_out/ev2/apply4_k1 python tools/apply_bench.py --synth --ks 1 --reps 3 > gpurun_out/ev2/ncu_apply1.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > gpurun_out/ev2/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev2/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > gpurun_out/ev2/ncu_bench.log 2>&1
echo done
ls gpurun_out/ev2
