# CUDA-graph replay of pdg_step(K) against the plain call
# (ran with the since-removed --graph flag; pdg_step replays its step graph by default now)
set -x
for c in 1 2 3; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2o_cfg$c.json 2>&1
done
