# config 2 with the persistent bulk-copy fused pass (one CTA per SM) instead of the register-staged kernel
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t2_pytest.log 2>&1; echo "pytest rc=$?"
for rep in 1 2; do
  timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/t2_cfg2_$rep.json 2>&1
  timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-tma > gpurun_out/t2_cfg2_notma_$rep.json 2>&1
done
for f in gpurun_out/t2_*.json; do echo "$f $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], {k:round(v['ms_total']/v['launches']*1e3,2) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; done
tail -3 gpurun_out/t2_pytest.log
