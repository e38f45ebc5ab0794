# config 2 with 3 CTAs per SM for the 2-D fused pass and the tiled sweep
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider \
    > gpurun_out/r2g_quick.log 2>&1; rc=$?; echo "quick rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
for c in 1 2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2g_cfg$c.json 2>&1
done
timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2g_cfg2b.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"relax_xsweep|sweep_cols" -s 6 -c 2 \
    -o gpurun_out/r2g_ncu_cfg2 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2g_ncu_cfg2.log 2>&1
echo "ncu rc=$?"
