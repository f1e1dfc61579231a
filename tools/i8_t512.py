import os, sys, numpy as np, torch
sys.path.insert(0, '.')
os.environ["EXPMB_I8"] = "1"
import paper_2512_20777_b200 as X
W = torch.as_tensor((np.random.default_rng(0).standard_normal((1, 512, 512)) / 22).astype(np.float32), device="cuda")
r = X.expm(W, 2.0 ** -24)
torch.cuda.synchronize()
print("ok", r.plan.m.tolist(), r.plan.s.tolist())
