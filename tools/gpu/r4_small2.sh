# small-problem kernel: parity and config 1 against PDG_NO_SMALL
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider > gpurun_out/m5_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/m5_pytest.log
for rep in 1 2; do
  for o in "" "--no-small"; do
    timeout 600 python bench.py --config 1 --steps 10 --warmup 5 --no-e2e --no-cpu-baseline $o > gpurun_out/m5_cfg1${o}_$rep.json 2>&1
  done
done
for f in gpurun_out/m5_*.json; do echo "$f $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], {k:(round(v['ms_total']/v['launches']*1e3,2), v['launches']) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; done
