# build, GPU suite (default and checked builds), default bench, config-2 bench + ncu of its two kernels,
# full-size parity of configs 2 and 3 as written
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"
PDG_CHECKED=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r2d_pytest_checked.log 2>&1; echo "pytest checked rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --config 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2d_cfg2.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"relax_xsweep|sweep_strided" -s 10 -c 2 \
    -o gpurun_out/r2d_ncu_cfg2 python bench.py --config 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2d_ncu_cfg2.log 2>&1
echo "ncu rc=$?"
bash tools/gpu/parity_long.sh cfg2,cfg3 1200
