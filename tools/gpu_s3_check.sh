# third-session check of the restored tree: GPU tests, smoke, bench, K2 dense-product timing
set -x
mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s3/smi.txt 2>&1
python tools/k2_bench.py > gpurun_out/s3/k2_bench.txt 2>&1; python tools/k2_bench.py --cols 34 >> gpurun_out/s3/k2_bench.txt 2>&1
python bench.py > gpurun_out/s3/bench.json 2> gpurun_out/s3/bench.err; echo bench rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/s3/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s3/gputests.log 2>&1; echo gputests rc=$?; tail -3 gpurun_out/s3/gputests.log
tail -c 600 gpurun_out/s3/bench.json
