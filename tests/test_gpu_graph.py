"""GPU: the fused training step captured in a CUDA graph (ops.TrainStepGraph, NEXT-2) replays
the same image, loss and gradients as direct calls, also after new inputs are copied in."""
import numpy as np
import pytest

import gsr_synth as S

pytestmark = pytest.mark.gpu


def test_train_step_graph_replay_matches_direct():
    import torch
    import paper_2501_06838_b200 as gsr
    from paper_2501_06838_b200 import ops
    P, m, scales = 16, 16, [1.7, 3.0, 4.0]
    n1 = m * P * P
    lay = gsr.layout([gsr.Image(P, P, s, k * n1, n1) for k, s in enumerate(scales)])
    n = n1 * len(scales)
    step = gsr.TrainStepGraph(lay, n)
    for seed in (1, 2):
        rng = np.random.default_rng(seed)
        raw = [rng.normal(-3, 1, n), rng.uniform(-0.5, 0.5, (n, 2)),
               np.concatenate([S.reference_grid(P, P, m)] * len(scales)),
               rng.normal(-0.5, 0.5, (n, 2)), rng.normal(0, 0.5, n), rng.normal(0, 1, (n, 3))]
        args = [torch.from_numpy(np.asarray(a, np.float32)).cuda() for a in raw]
        gt = torch.rand(lay.out_numel, device="cuda")
        out_d, loss_d, g_d = ops.train_step_l1(*args, lay, gt)
        out_d, loss_d = out_d.clone(), loss_d.clone()
        g_d = {k: v.clone() for k, v in g_d.items()}
        out_g, loss_g, g_g = step(*args, gt)
        torch.cuda.synchronize()
        assert torch.allclose(out_g, out_d, rtol=1e-6, atol=1e-7)
        assert abs(loss_g.item() - loss_d.item()) <= 1e-9 * abs(loss_d.item())
        for k in g_d:
            scale = g_d[k].abs().max().item() + 1e-30
            assert (g_g[k] - g_d[k]).abs().max().item() <= 1e-5 * scale, k
