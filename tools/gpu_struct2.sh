# full GPU suite after the structured butterfly black box + column-run fix
set -x
mkdir -p gpurun_out/st2
timeout 2700 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/st2/gputests.log 2>&1; echo gputests rc=$?; tail -5 gpurun_out/st2/gputests.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "structured" -p no:cacheprovider 2>&1 | grep "vr=" > gpurun_out/st2/struct.log; cat gpurun_out/st2/struct.log
