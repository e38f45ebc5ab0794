# pdg_step as a replayed CUDA graph: full suite + small configs with and without
set -x
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2p_pytest.log 2>&1; rc=$?; echo "pytest rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
python - > gpurun_out/r2p_graph_timing.txt 2>&1 <<'P'
import torch, time, sys
sys.path.insert(0, '.')
from paper_1702_00169_b200 import pdg
from pdg_inputs import CONFIGS, w0_grid
for key, steps in ((1, 100), (2, 100), (3, 50)):
    cfg = CONFIGS[key]
    for flags in (0, pdg.PDG_NO_GRAPH):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            S = pdg.Solver(pdg.problem_from_config(cfg, flags=flags))
            S.set_equilibrium(w0_grid(cfg, device='cuda').reshape(-1))
            S.step(steps)  # warm (captures the graph)
            st.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st); S.step(steps); e1.record(st); st.synchronize()
            print(f"config {key} flags {flags}: {e0.elapsed_time(e1) / steps * 1e3:.2f} us per step")
            S.destroy()
P
cat gpurun_out/r2p_graph_timing.txt
