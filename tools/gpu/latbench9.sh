for L in D3Q19 D3Q27; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat9_$L.json 2> gpurun_out/lat9_$L.err; done
timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat9_D2Q9.json 2>&1
cp paper_1702_00169_b200/libpdg_mmaall.so paper_1702_00169_b200/libpdg.so
timeout 600 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_source.py -q -x 2>&1 | tail -3
for L in D3Q19 D3Q27; do timeout 600 python bench.py --lattice $L --cells 128 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat9m_$L.json 2> gpurun_out/lat9m_$L.err; done
timeout 600 python bench.py --lattice D2Q9 --cells 1024 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lat9m_D2Q9.json 2>&1
echo done
