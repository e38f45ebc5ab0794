set -x
export OMP_NUM_THREADS=12   # t2_all runs the 24 velocities in 2 rounds either way; bounds the fold copies (config 5)
bash tools/gpu/parity_long.sh cfg4,cfg4s 4500
