PAQIF_NVCC_EXTRA=-DPAQIF_TVD_PROF python -c "from paper_2008_03276_b200 import build; build.build(force=True)"
python - <<'PY'
import numpy as np
from paper_2008_03276_b200.tvdcd import KappaSchemeConfig, quartic_test_problem, sweep_splitting
prob, _ = quartic_test_problem(512, KappaSchemeConfig(kappa=1/3, eps=1e-6))
sweep_splitting(prob, np.zeros_like(prob.f), "Ls1")
import torch; torch.cuda.synchronize()
PY
