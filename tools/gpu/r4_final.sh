# round-2 closing evidence (small-problem kernel, oracle aliasing fix, conditioning-aware fuzz bars): build + smoke, the GPU suite (widened fuzz) with the default and the
# checked builds, the default bench twice, the reference arm, a 1-rank torchrun launch, configs
# 2-4 and the lattice workloads, the ncu launch list of the default bench command and --set full
# captures of its two kernels
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/g4_smoke.log 2>&1; echo "smoke rc=$?"
python -m paper_1702_00169_b200.build --checked > /dev/null 2>&1
PDG_FUZZ_SEEDS_MAIN=400 PDG_FUZZ_SEEDS_BACKWARD=400 PDG_FUZZ_SEEDS=200 timeout 2400 python -m pytest tests -m gpu -q \
    -p no:cacheprovider -rs > gpurun_out/g4_pytest.log 2>&1; echo "pytest rc=$?"
PDG_CHECKED=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/g4_pytest_checked.log 2>&1
echo "pytest checked rc=$?"
for k in 1 2; do timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/g4_bench_$k.json 2> gpurun_out/g4_bench_$k.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/g4_ref.json 2> gpurun_out/g4_ref.err; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g4_torchrun1.json 2> gpurun_out/g4_torchrun1.err
echo "torchrun rc=$?"
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/g4_cfg$c.json 2>&1
done
for L in D3Q15 D3Q19 D3Q27; do
  timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g4_lat_$L.json 2>&1
done
timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g4_lat_D2Q9.json 2>&1
CMD="python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/g4_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"sweep|relax|zslab|lattice|equilibrium|check_state" -c 200 --csv \
    --log-file gpurun_out/g4_launches.csv $CMD > gpurun_out/g4_ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"relax_xsweep_kernel" -s 1 -c 1 \
    -o gpurun_out/g4_ncu_relax $CMD > gpurun_out/g4_ncu_relax.log 2>&1; echo "ncu relax rc=$?"
python tools/ncu_full_summary.py gpurun_out/g4_ncu_relax.ncu-rep > gpurun_out/g4_ncu_relax.txt 2>&1 && rm -f gpurun_out/g4_ncu_relax.ncu-rep
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"sweep_strided_kernel" -s 4 -c 1 \
    -o gpurun_out/g4_ncu_strided $CMD > gpurun_out/g4_ncu_strided.log 2>&1; echo "ncu strided rc=$?"
python tools/ncu_full_summary.py gpurun_out/g4_ncu_strided.ncu-rep > gpurun_out/g4_ncu_strided.txt 2>&1 && rm -f gpurun_out/g4_ncu_strided.ncu-rep
# config 2 with the L2 policy: the two kernels of a step without ncu's cache flush (--cache-control none),
# so the dram vs lts split shows f staying in L2 between the passes
CMD2="python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct \
    --cache-control none --clock-control none -k regex:"sweep_cols|relax_xsweep" -s 8 -c 4 --csv \
    --log-file gpurun_out/g4_cfg2_l2.csv $CMD2 > gpurun_out/g4_cfg2_l2.log 2>&1; echo "ncu cfg2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_cols|relax_xsweep" -s 8 -c 2 \
    -o gpurun_out/g4_ncu_cfg2 $CMD2 > gpurun_out/g4_ncu_cfg2.log 2>&1; echo "ncu cfg2 full rc=$?"
python tools/ncu_full_summary.py gpurun_out/g4_ncu_cfg2.ncu-rep > gpurun_out/g4_ncu_cfg2.txt 2>&1
ncu -i gpurun_out/g4_ncu_cfg2.ncu-rep --page details --csv > gpurun_out/g4_ncu_cfg2_details.csv 2>&1 && rm -f gpurun_out/g4_ncu_cfg2.ncu-rep
du -sh gpurun_out
for f in gpurun_out/g4_*.json; do echo "$f $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d.get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'))" 2>&1 | tail -1)"; done
