# programmatic dependent launches: parity (PDL vs plain order vs oracle) and A/B benches
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
    -k "programmatic or graph_replay or resynced or stabilised or profile_pause" > gpurun_out/p4_pytest.log 2>&1; echo "pytest rc=$?"
for rep in 1 2; do
  for c in 1 2 3; do
    for o in "" "--no-pdl"; do
      timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $o > gpurun_out/p4_cfg${c}${o}_$rep.json 2>&1
    done
  done
done
for o in "" "--no-pdl"; do
  timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $o > gpurun_out/p4_cfg4${o}.json 2>&1
  timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $o > gpurun_out/p4_cfg5${o}.json 2>&1
  timeout 600 python bench.py --lattice D3Q19 --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $o > gpurun_out/p4_latD3Q19${o}.json 2>&1
done
grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/p4_*.json | head -0
for f in gpurun_out/p4_*.json; do echo "$f $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"; done
tail -3 gpurun_out/p4_pytest.log
