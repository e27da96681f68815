# fourth round-2 session: evidence re-run on the committed tree
set -x
mkdir -p gpurun_out/fin4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/fin4/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/fin4/gputests.log 2>&1; echo gputests rc=$?; tail -3 gpurun_out/fin4/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin4/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/fin4/smoke.log
python bench.py > gpurun_out/fin4/bench.json 2> gpurun_out/fin4/bench.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/fin4/bench_ref.json 2> gpurun_out/fin4/bench_ref.err; echo ref rc=$?
python tools/run_configs.py --cfg 0 1 2 4 --reps 4 > gpurun_out/fin4/configs.log 2>&1
python tools/run_configs.py --cfg 4 --reps 3 --c64 > gpurun_out/fin4/cfg4_c64.log 2>&1
python tools/run_configs.py --cfg 3 --n 16384 --reps 2 > gpurun_out/fin4/cfg3_16384.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin4/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > gpurun_out/fin4/ncu_bench.log 2>&1; echo ncu rc=$?
tail -c 800 gpurun_out/fin4/bench.json
