"""Small invocations of each hand-written kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py <case>

cases: c2 (3xTF32 warp kernel), c1 (DMMA fused), i8 (int8-slice tcgen05 stage),
tile (fused one-CTA-per-matrix, n = 96), gemm (bucketed pipeline, n = 200 fp64),
lowrank (DMMA warp kernel + t > 32 path), select (plan only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_20777_b200 as X  # noqa: E402


def main(case):
    torch.manual_seed(0)
    if case == "c2":
        W = torch.randn(64, 16, 16, device="cuda")
        W = (W - W.transpose(-1, -2)) / 8
        X.expm(W, 2.0 ** -24)
    elif case == "c1":
        X.expm(torch.randn(4, 64, 64, device="cuda", dtype=torch.float64) / 20, 2.0 ** -53)
    elif case == "i8":
        X.expm(torch.randn(2, 512, 512, device="cuda") / 8, 2.0 ** -24)
    elif case == "tile":
        X.expm(torch.randn(3, 96, 96, device="cuda", dtype=torch.float64) / 5, 1e-12)
        X.expm(torch.randn(3, 96, 96, device="cuda") / 5, 2.0 ** -24)
    elif case == "gemm":
        X.expm(torch.randn(2, 200, 200, device="cuda", dtype=torch.float64) / 5, 1e-12)
    elif case == "lowrank":
        a1 = torch.rand(8, 64, 8, device="cuda", dtype=torch.float64) - 0.5
        a2 = (torch.rand(8, 8, 64, device="cuda", dtype=torch.float64) - 0.5) / 8
        X.expm_lowrank(X.LowRankPair(a1, a2), 1e-12)
        b1 = torch.rand(2, 80, 40, device="cuda", dtype=torch.float64) - 0.5
        b2 = (torch.rand(2, 40, 80, device="cuda", dtype=torch.float64) - 0.5) / 40
        X.expm_lowrank(X.LowRankPair(b1, b2), 1e-12)
    elif case == "select":
        X.select_sastre(torch.randn(16, 32, 32, device="cuda", dtype=torch.float64) / 3, 1e-12)
    torch.cuda.synchronize()
    print("ok", case)


if __name__ == "__main__":
    main(sys.argv[1])
