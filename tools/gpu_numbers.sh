# round-2 numbers: bench line, every config's construction, apply sweeps, FP64/FP32 peaks
mkdir -p gpurun_out/num
./tools/microbench/fp64_peaks > gpurun_out/num/peaks.txt 2>&1
python bench.py > gpurun_out/num/bench.json 2> gpurun_out/num/bench.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/num/bench_ref.json 2> gpurun_out/num/bench_ref.err; echo ref rc=$?
python tools/run_configs.py --cfg 0 1 2 4 --reps 4 > gpurun_out/num/configs.log 2>&1
python tools/run_configs.py --cfg 4 --reps 3 --c64 > gpurun_out/num/cfg4_c64.log 2>&1
python tools/run_configs.py --cfg 3 --n 4096 --reps 2 --profile > gpurun_out/num/cfg3_4096.log 2>&1
python tools/run_configs.py --cfg 3 --n 16384 --reps 1 --profile > gpurun_out/num/cfg3_16384.log 2>&1
python tools/apply_bench.py --synth --ks 1,2,8,16,32,66 --reps 20 > gpurun_out/num/apply_cfg4.log 2>&1
python tools/apply_bench.py --cfg 2 --ks 1,2,8,16,32 --reps 20 > gpurun_out/num/apply_cfg2.log 2>&1
tail -c 600 gpurun_out/num/bench.json; cat gpurun_out/num/peaks.txt | head -4
