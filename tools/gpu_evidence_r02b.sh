# round-2 (second session) evidence: K2 full capture, cpqr_warp capture, launch list, bench (both arms)
set -x
mkdir -p gpurun_out/ev
python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/ev/cfg2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:matvec_oz -s 8 -c 1 -o gpurun_out/ev/k2 python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/ev/ncu_k2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cpqr_warp -s 6 -c 1 -o gpurun_out/ev/cpqr_warp python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/ev/ncu_cpqr.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > gpurun_out/ev/bench_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > gpurun_out/ev/ncu_launch.log 2>&1
python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err; echo ref rc=$?
python tools/k2_bench.py > gpurun_out/ev/k2_bench.txt 2>&1
ls -la gpurun_out/ev
