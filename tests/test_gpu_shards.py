"""One-GPU check of the multi-GPU decomposition: ``expm`` of
a full batch is bit-identical to the rank-ordered concatenation of ``expm``
over the ``shard_range(r, world, B)`` slices -- what N ranks compute and the
final gather brings home -- for world in {2, 4, 8}, on the fused small-n
kernels (n = 16, 64), the FFMA/DMMA GEMM pipeline (n = 256) and the exact
int8-slice tensor-core path (fp32 n = 2048).  The reference's analogue:
parallel == serial (tests/test_bench.py:165-173, bench.py:303-309)."""
import numpy as np
import pytest
import torch

import paper_2512_20777_b200 as X
from paper_2512_20777_b200.shard import shard_range

pytestmark = pytest.mark.gpu


def _batch(n, B, dtype, seed):
    g = torch.Generator().manual_seed(seed)
    W = torch.randn(B, n, n, generator=g, dtype=torch.float64)
    W *= (10.0 ** (torch.rand(B, generator=g, dtype=torch.float64) * 3 - 1.5)
          / W.abs().sum(dim=-2).amax(dim=-1))[:, None, None]
    return W.to(dtype).cuda()


@pytest.mark.parametrize("n,B,dtype", [(16, 1000, torch.float32), (64, 300, torch.float64),
                                       (256, 40, torch.float32), (256, 24, torch.float64),
                                       (2048, 8, torch.float32)])
def test_shards_concat_bit_identical(n, B, dtype):
    W = _batch(n, B, dtype, seed=n + B)
    eps = 2.0 ** -24 if dtype == torch.float32 else 2.0 ** -53
    full = X.expm(W, eps)
    for world in (2, 4, 8):
        parts = [X.expm(W[a:b].clone(), eps) for a, b in (shard_range(r, world, B) for r in range(world))
                 if b > a]
        val = torch.cat([p.value for p in parts])
        assert torch.equal(val, full.value), (n, world)
        assert torch.equal(torch.cat([p.plan.m for p in parts]), full.plan.m)
        assert torch.equal(torch.cat([p.plan.s for p in parts]), full.plan.s)
        assert torch.equal(torch.cat([p.mults for p in parts]), full.mults)
