# Full-size parity protocol (tests/test_gpu_long.py) for the cases named in $1 (comma-separated,
# e.g. cfg2,cfg3,cfg2s,cfg3s); records in gpurun_out/parity/, the pytest log next to them.
set -x
mkdir -p gpurun_out/parity
python -c "import __graft_entry__ as g; g.build()" || exit 1
PDG_PARITY_LONG=1 PDG_PARITY_CASES="$1" PDG_PARITY_OUT=gpurun_out/parity \
    timeout ${2:-5400} python -m pytest tests/test_gpu_long.py -q -s -p no:cacheprovider -rs \
    > gpurun_out/parity/pytest_$(echo $1 | tr ',' '_').log 2>&1
echo "pytest rc=$?"
free -g > gpurun_out/parity/free_$(echo $1 | tr ',' '_').txt
