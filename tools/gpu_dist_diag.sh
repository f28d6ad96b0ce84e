#!/bin/bash
python tools/gpu_dist_diag.py single 0
AIFMM_NULLSPACE=0 python tools/gpu_dist_diag.py single_nons 0
AIFMM_DIST_FORCE=1 python tools/gpu_dist_diag.py w1 1
python tools/gpu_dist_diag.py w2 2
AIFMM_DIST_PHASES=1 python tools/gpu_dist_diag.py w2_cmp 2
AIFMM_DIST_PHASES=2 python tools/gpu_dist_diag.py w2_piv 2
AIFMM_DIST_PHASES=4 python tools/gpu_dist_diag.py w2_schur 2
python - <<'PY'
import numpy as np
X = {t: np.load(f"gpurun_out/x_{t}.npy") for t in ["single", "single_nons", "w1", "w2", "w2_cmp", "w2_piv", "w2_schur"]}
R = {t: np.load(f"gpurun_out/ranks_{t}.npz") for t in X}
ref = X["single_nons"]
for t, x in X.items():
    mism = {l: int(np.sum(R[t][l] != R["single_nons"][l])) for l in R[t].files}
    print(t, "rel vs single_nons %.2e" % (np.linalg.norm(x - ref) / np.linalg.norm(ref)), "vs single %.2e" % (np.linalg.norm(x - X["single"]) / np.linalg.norm(X["single"])), "rank mismatches", mism)
PY
