# source-level stall attribution of the body-diagonal lattice sweep (D3Q15 128^3): ncu --set full with source
set -x
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"lattice_sweep_kernel<\(int\)3, \(int\)3, \(int\)7" -s 2 -c 1 -o gpurun_out/l4_act7 \
    python bench.py --lattice D3Q15 --cells 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/l4_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/l4_act7.ncu-rep --page source --csv > gpurun_out/l4_src_cuda.csv 2> gpurun_out/l4_src_err.txt
ncu -i gpurun_out/l4_act7.ncu-rep --page source --csv --print-source sass > gpurun_out/l4_src_sass.csv 2>> gpurun_out/l4_src_err.txt
python tools/ncu_full_summary.py gpurun_out/l4_act7.ncu-rep > gpurun_out/l4_summary.txt 2>&1
ls -la gpurun_out/l4_*
rm -f gpurun_out/l4_act7.ncu-rep
