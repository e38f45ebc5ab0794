# aligned warp sweeps (compile-time chunking when the line is a multiple of 32 K cells) in the fused
# pass and the tile kernel; one tile per CTA in sweep_cols: parity + configs 2-5
set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/a3_pytest.log 2>&1; echo "pytest rc=$?"
for c in 2 3 4; do for k in 1 2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/a3_cfg${c}_$k.json 2>&1
done; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/a3_cfg5.json 2>&1
CMD="python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_cols|relax_xsweep" -s 8 -c 2 \
    -o gpurun_out/a3_ncu_cfg2 $CMD > gpurun_out/a3_ncu.log 2>&1; echo "ncu rc=$?"
