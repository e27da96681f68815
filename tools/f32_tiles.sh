for t in 0 1 2 3 4; do echo "tile $t"; BFLY_F32_TILE=$t python tools/run_configs.py --cfg 4 --reps 2 --profile --c64 2>&1 | grep "kernel bgemm_f32\|cfg"; done
echo default; python tools/run_configs.py --cfg 4 --reps 2 --profile --c64 2>&1 | grep "kernel bgemm_f32\|cfg"
