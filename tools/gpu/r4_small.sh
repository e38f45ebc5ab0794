# small-problem kernel (one CTA, f in shared memory): parity, full suite, config 1 bench against PDG_NO_SMALL
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "small_problem or config1 or composed or graph_replay or profile_pause" > gpurun_out/m4_pytest_small.log 2>&1; echo "pytest small rc=$?"
tail -n 3 gpurun_out/m4_pytest_small.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/m4_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/m4_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m4_smoke.log 2>&1; echo "smoke rc=$?"
for rep in 1 2; do
  timeout 600 python bench.py --config 1 --steps 10 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/m4_cfg1_$rep.json 2>&1
done
for f in gpurun_out/m4_*.json; do echo "$f $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], {k:(round(v['ms_total']/v['launches']*1e3,2), v['launches']) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; done
