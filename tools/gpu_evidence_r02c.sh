# pair-kernel capture + bench after the CTA-pair and exponent-add changes
mkdir -p gpurun_out/ev3
python tools/run_configs.py --cfg 2 --reps 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:matvec_oz_pair -c 1 -o gpurun_out/ev3/k2pair python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/ev3/ncu_pair.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:matvec_oz_kernel -s 4 -c 1 -o gpurun_out/ev3/k2 python tools/run_configs.py --cfg 2 --reps 1 > gpurun_out/ev3/ncu_k2.log 2>&1
python bench.py > gpurun_out/ev3/bench.json 2> gpurun_out/ev3/bench.err; echo bench rc=$?
python tools/k2_bench.py > gpurun_out/ev3/k2_bench.txt 2>&1; python tools/k2_bench.py --cols 34 >> gpurun_out/ev3/k2_bench.txt 2>&1
ls gpurun_out/ev3
