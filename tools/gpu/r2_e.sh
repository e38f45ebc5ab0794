# full-size parity of config 5 and its stabilised twin (oracle on the host, 12 threads: the 24
# velocities of a T2 run in two rounds either way; bounds the per-velocity copies), then the
# oracle's single-thread / all-core table of configs 1-3
set -x
export OMP_NUM_THREADS=12
bash tools/gpu/parity_long.sh cfg5,cfg5s 4800
unset OMP_NUM_THREADS
timeout 1200 python bench.py --oracle-table > gpurun_out/r2e_oracle_table.json 2> gpurun_out/r2e_oracle_table.err; echo "oracle table rc=$?"
