import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from oracle import oracle as O
from paper_1702_00169_b200 import pdg
from pdg_inputs import CONFIGS
from gpu_helpers import rel_maxnorm, to_np
import test_gpu_parity as T
for key, N, sch, tau, steps in [(4,1,"m2kin",0.01,4),(4,1,"m2",0.0,1),(4,2,"m2",0.0,1),(3,1,"m2",0.0,1),(4,1,"m2kin",0.0,1)]:
    code = {"m2": pdg.PDG_SCHEME_M2, "m2kin": pdg.PDG_SCHEME_M2KIN}[sch]
    cfg = CONFIGS[key].resized(N).stabilised()
    pb, f0, fbg = T.seeded_equilibrium(cfg); pb.tau = tau
    ref = O.scheme_run(pb, f0, fbg, steps, sch)
    r = []
    for flags in (0, pdg.PDG_NO_SMALL):
        S = T.gpu_with_state(cfg, f0, fbg, scheme=code, tau=tau, flags=flags)
        S.step(steps); got = to_np(S.get_state(), f0.shape); S.destroy()
        err = np.abs(got - ref).reshape(got.shape[0], -1).max(axis=1) / np.abs(ref).max()
        r.append((rel_maxnorm(got, ref), np.nonzero(err > 1e-12)[0].tolist()))
    print(key, N, sch, tau, steps, r, flush=True)
