# round-2 evidence re-run on the committed tree: GPU tests, bench (both arms), config/apply sweeps, peaks
set -x
mkdir -p gpurun_out/fin
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/fin/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/fin/gputests.log 2>&1; echo gputests rc=$?; tail -3 gpurun_out/fin/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/fin/smoke.log
python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/fin/bench_ref.json 2> gpurun_out/fin/bench_ref.err; echo ref rc=$?
./tools/microbench/fp64_peaks > gpurun_out/fin/peaks.txt 2>&1
python tools/run_configs.py --cfg 0 1 2 4 --reps 4 > gpurun_out/fin/configs.log 2>&1
python tools/run_configs.py --cfg 4 --reps 3 --c64 > gpurun_out/fin/cfg4_c64.log 2>&1
python tools/apply_bench.py --synth --ks 1,2,4,8,16,32,66 --reps 20 > gpurun_out/fin/apply_cfg4.log 2>&1
python tools/apply_bench.py --cfg 2 --ks 1,2,8,16,32 --reps 20 > gpurun_out/fin/apply_cfg2.log 2>&1
tail -c 1500 gpurun_out/fin/bench.json
