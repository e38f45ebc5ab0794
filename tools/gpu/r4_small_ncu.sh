# ncu --set full of the small-problem kernel (config 1, ten steps in one launch)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"small_run" -s 2 -c 1 -o gpurun_out/sm_ncu \
    python bench.py --config 1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sm_ncu.log 2>&1
echo "ncu rc=$?"
python tools/ncu_full_summary.py gpurun_out/sm_ncu.ncu-rep > gpurun_out/sm_summary.txt 2>&1
ncu -i gpurun_out/sm_ncu.ncu-rep --page source --csv --print-source sass > gpurun_out/sm_src.csv 2>/dev/null
rm -f gpurun_out/sm_ncu.ncu-rep
cat gpurun_out/sm_summary.txt
