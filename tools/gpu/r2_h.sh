# round-2 ncu evidence of the headline: launch list of the default bench command and a --set full
# capture of its two kernels (config 5), plus the launch list of the 8-slab z-slab emulation
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/r2h_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2h_launches.csv $CMD > gpurun_out/r2h_ncu_launches.log 2>&1
echo "launch list rc=$?"
CMDZ="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --decomp zslab --slabs-per-rank 8"
$CMDZ > gpurun_out/r2h_plainz.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2h_launches_zslab8.csv $CMDZ > gpurun_out/r2h_ncu_launchesz.log 2>&1
echo "launch list z rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"relax_xsweep|sweep_strided" -s 2 -c 2 \
    -o gpurun_out/r2h_ncu_full_cfg5 $CMD > gpurun_out/r2h_ncu_full.log 2>&1
echo "ncu full rc=$?"
