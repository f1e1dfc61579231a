#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/prec.py <<'PY'
import numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2512_20777_b200 as X
from paper_2512_20777_b200 import workloads as WL
from oracle import expm_oracle as O
W = WL.generate("C2")
val, m, s, *_ = O.expm_batch(W[:16384].astype(np.float64), 2.0**-24)
for v in ("1", "2"):
    os.environ["EXPMB_VARIANT"] = v
PY
for v in 1 2; do EXPMB_VARIANT=$v python - <<'PY'
import numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2512_20777_b200 as X
from paper_2512_20777_b200 import workloads as WL
from oracle import expm_oracle as O
W = WL.generate("C2", batch=16384)
val, m, s, *_ = O.expm_batch(W.astype(np.float64), 2.0**-24)
r = X.expm(torch.as_tensor(W).cuda(), 2.0**-24).value.double().cpu().numpy()
err = np.abs(r - val).sum(axis=1).max(axis=1) / np.abs(val).sum(axis=1).max(axis=1)
print(os.environ["EXPMB_VARIANT"], "worst", err.max(), "mean", err.mean(), "p99", np.quantile(err, 0.99))
PY
done > gpurun_out/prec.txt 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:expm_fused -s 3 -c 1 -o gpurun_out/prof_C2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
