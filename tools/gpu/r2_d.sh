# build, quick check of the new kernels, GPU suite (default and checked builds), default bench with and
# without TMA staging, config-2 bench + ncu of its two kernels, full-size parity of configs 2 and 3
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python -m pytest tests/test_gpu_bench_kernels.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
    > gpurun_out/r2d_quick.log 2>&1; rc=$?; echo "quick rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "bench rc=$?"
for c in 2 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2d_cfg$c.json 2>&1
done
timeout 600 python bench.py --no-tma --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2d_bench_notma.json 2>&1
for c in 2 3 4; do
  timeout 600 python bench.py --no-tma --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2d_cfg${c}_notma.json 2>&1
done
PDG_CHECKED=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r2d_pytest_checked.log 2>&1; echo "pytest checked rc=$?"
timeout 300 python bench.py --config 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2d_cfg2_100.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"relax_xsweep|sweep_cols" -s 10 -c 2 \
    -o gpurun_out/r2d_ncu_cfg2 python bench.py --config 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2d_ncu_cfg2.log 2>&1
echo "ncu rc=$?"
bash tools/gpu/parity_long.sh cfg2,cfg3 1200
