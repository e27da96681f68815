# apply timings: config-4 input butterfly (k = 1..66) and config-2 factorization (k = 1, 2, 16)
python tools/apply_bench.py --synth --ks 1,8,16,32,66 --reps 20 2>&1 | tail -5
python tools/apply_bench.py --cfg 2 --ks 1,2,8,16 --reps 20 2>&1 | tail -4
