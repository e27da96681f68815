# K2 diagonal set: e >= 5 (default build) vs e >= 4 (round 2, libbfly_b200_e4.so): parity + same-box A/B
mkdir -p gpurun_out/e5
timeout 1500 python -m pytest tests/test_full_parity.py tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/e5/parity.log 2>&1; echo parity rc=$?; tail -3 gpurun_out/e5/parity.log
bash tools/k2_ab.sh paper_2002_03400_b200/_native/libbfly_b200.so paper_2002_03400_b200/_native/libbfly_b200_e4.so > gpurun_out/e5/ab.txt 2>&1; cat gpurun_out/e5/ab.txt
python tools/run_configs.py --cfg 0 1 2 4 --reps 3 > gpurun_out/e5/configs.log 2>&1; grep "^cfg" gpurun_out/e5/configs.log
