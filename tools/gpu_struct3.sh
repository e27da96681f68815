# output-restricted structured black box: tests, projected scaling (config 4), bench
set -x
mkdir -p gpurun_out/st3
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_multiprocess.py -m gpu -q -x -s -k "structured or virtual_ranks or multiprocess or two_process" -p no:cacheprovider > gpurun_out/st3/tests.log 2>&1; echo tests rc=$?; tail -6 gpurun_out/st3/tests.log
BFLY_POOL_RESERVE_GB=100 python tools/project_scaling.py --cfg 4 --reps 3 > gpurun_out/st3/proj4.txt 2> gpurun_out/st3/proj4.err; echo rc=$?; grep -v phases gpurun_out/st3/proj4.txt | head
python bench.py > gpurun_out/st3/bench.json 2> gpurun_out/st3/bench.err; echo bench rc=$?
tail -c 1500 gpurun_out/st3/bench.json
