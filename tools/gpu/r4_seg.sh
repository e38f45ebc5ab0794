# segment_passes with the off-chain inflow correction: parity of the axis-aligned sweeps, benches of configs 1-5
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_kernels.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider > gpurun_out/s4_pytest.log 2>&1; echo "pytest rc=$?"
for rep in 1 2; do
  for c in 1 2 3; do
    timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/s4_cfg${c}_$rep.json 2>&1
  done
done
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4_cfg4.json 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4_cfg5.json 2>&1
for f in gpurun_out/s4_*.json; do echo "$f $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], {k:round(v['ms_total']/v['launches']*1e3,2) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; done
tail -3 gpurun_out/s4_pytest.log
