import torch, paper_2512_20777_b200 as ex
W = torch.randn(65536, 16, 16, device="cuda")          # fp32 or fp64, [..., n, n]
res = ex.expm(W, 2.0 ** -24)                           # scheme="sastre" | "ps"
res.value, res.plan.m, res.plan.s, res.plan.e1, res.plan.e2, res.mults
ex.expm_baseline(W, 2.0 ** -24)                        # Alg. 1 (engine.py:90-116), n <= 64
ex.expm_host(W.cpu().pin_memory(), 2.0 ** -24)         # host buffers in/out, pipelined copies
A1 = torch.randn(4096, 64, 8, device="cuda", dtype=torch.float64) / 8   # W = A1 A2, rank 8
A2 = torch.randn(4096, 8, 64, device="cuda", dtype=torch.float64) / 8
ex.expm_lowrank(ex.LowRankPair(A1, A2), 1e-12)         # I + A1 psi(A2 A1) A2 (engine.py:198-257)
A = torch.randn(256, 256, device="cuda") / 16
ex.expm_timegrid(A, torch.linspace(0, 4, 4096), 2.0 ** -24)   # e^(t_k A), shared powers

print('readme examples ok', res.value.shape)
