"""GPU parity of the NEXT-1 fused training step (gsr_train_step_l1_batched) against the float64
oracle composition (oracle/train.py): activations -> render -> L1 loss -> raw gradients."""
import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from oracle import train as T
from _util import assert_fwd_close

pytestmark = pytest.mark.gpu

RAWK = ("raw_alpha", "offset", "raw_sigma", "raw_rho", "raw_color")


def raw_cloud(H, W, seed, m=16):
    """Raw head outputs with the image-like distribution of gsr_synth (before activation)."""
    rng = np.random.default_rng(seed)
    n = m * H * W
    ref = S.reference_grid(H, W, m).astype(np.float32)
    raw = dict(raw_alpha=rng.normal(-3, 1, n), offset=rng.uniform(-0.5, 0.5, (n, 2)),
               raw_sigma=rng.normal(-0.5, 0.5, (n, 2)), raw_rho=rng.normal(0, 0.5, n),
               raw_color=rng.normal(0, 1, (n, 3)))
    return {k: v.astype(np.float32) for k, v in raw.items()}, ref


def gt_near(I, seed, delta=2e-3):
    """Ground truth offset from the oracle image by +-delta (no sign ties under fp32 error)."""
    rng = np.random.default_rng(seed)
    return (I + rng.choice([-delta, delta], size=I.shape)).astype(np.float32)


@pytest.mark.parametrize("rho_scale,scales", [
    (1.0, [4.0, 2.5, 1.3]), (1 - 1e-4, [4.0, 2.5, 1.3]),
    (1.0, [(4.0, 2.0), (2.5, 2.5), (1.3, 3.1)]),       # scale vectors (R22)
    (1.0, [12.5, 7.3])])                                 # HAT-L range s ~ U[1, 16]
def test_train_step_batch_matches_oracle(rho_scale, scales):
    import torch
    import paper_2501_06838_b200 as gsr
    from paper_2501_06838_b200 import ops
    raws, refs, imgs, gts = [], [], [], []
    off = 0
    for k, s in enumerate(scales):
        H, W = 20, 24
        raw, ref = raw_cloud(H, W, seed=50 + k)
        n = raw["raw_alpha"].shape[0]
        act = T.activate(raw, ref, rho_scale)
        gts.append(gt_near(O.render_fwd(act, H, W, s, 0.1), seed=k))
        raws.append(raw); refs.append(ref); imgs.append((H, W, s, off, n)); off += n
    raw = {k: np.concatenate([r[k] for r in raws]) for k in RAWK}
    ref = np.concatenate(refs)
    outs, loss, g = T.l1_step(raw, ref, imgs, gts, 0.1, rho_scale)
    lay = gsr.layout([gsr.Image(H, W, s[0], go, gc, s_y=s[1]) if isinstance(s, tuple) else
                      gsr.Image(H, W, s, go, gc) for (H, W, s, go, gc) in imgs])
    dev = {k: torch.from_numpy(v).cuda() for k, v in raw.items()}
    gt_flat = torch.from_numpy(np.concatenate([x.reshape(-1) for x in gts])).cuda()
    out, gl, gg = ops.train_step_l1(dev["raw_alpha"], dev["offset"], torch.from_numpy(ref).cuda(),
                                    dev["raw_sigma"], dev["raw_rho"], dev["raw_color"], lay, gt_flat,
                                    0.1, rho_scale)
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        assert_fwd_close(lay.view(out, k).cpu().numpy(), o)
    assert float(gl.item()) == pytest.approx(loss, rel=1e-5)
    cols = [("raw_alpha", [0]), ("offset", [1, 2]), ("raw_sigma", [3, 4]), ("raw_rho", [5]),
            ("raw_color", [6, 7, 8])]
    for name, c in cols:
        got = gg[name].cpu().numpy().astype(np.float64).reshape(len(ref), -1)
        want = np.asarray(g[name]).reshape(len(ref), -1)
        S_ = g["absmass"][:, c]
        bound = 1e-4 * np.maximum(np.abs(want), 0.1 * S_) + 1e-8 * S_.max(axis=0, keepdims=True)
        err = np.abs(got - want)
        assert (err <= bound + 1e-30).all(), (name, float((err / (bound + 1e-30)).max()))


@pytest.mark.parametrize("B,P,smax,seed", [(16, 48, 4.0, 3),     # EDSR/RDN slice
                                           (8, 64, 16.0, 4)])    # HAT-L slice
def test_train_step_real_shapes_and_graph(B, P, smax, seed):
    """NEXT-2: the fused training step at the paper's per-GPU training batch shapes (m = 16,
    per-patch s ~ U[1, smax]), launched directly and replayed from a CUDA graph
    (ops.TrainStepGraph), vs the float64 oracle composition: every image element, the loss,
    and the raw gradients of 64 sampled Gaussians per patch.

    The oracle activates in fp64 and rounds the render's inputs to float32 as the CUDA path
    does (reading R23: mu = ref + offset is the fp32 sum -- without it, mu's rounding alone
    moves narrow Gaussians' terms by ~2e-4 relative); the CUDA sigmoid/tanh are within ~3 ulp
    of the correctly rounded values, i.e. the render inputs still differ by a few fp32 ulp:
    forward gate 1e-5 + 2e-6 |I|; raw gradients at R18's 1e-1 S as in
    test_train_step_batch_matches_oracle."""
    import torch
    import paper_2501_06838_b200 as gsr
    from paper_2501_06838_b200 import ops
    rng = np.random.default_rng(seed)
    scales = rng.uniform(1.0, smax, B)
    raws, refs, imgs, gts, sample = [], [], [], [], []
    off = 0
    for k in range(B):
        raw, ref = raw_cloud(P, P, seed=1000 * seed + k)
        n = raw["raw_alpha"].shape[0]
        act = T.activate(raw, ref, 1.0, fp32=True)
        gts.append(gt_near(O.render_fwd(act, P, P, float(scales[k]), 0.1), seed=k))
        raws.append(raw); refs.append(ref); imgs.append((P, P, float(scales[k]), off, n))
        sample.append(np.sort(rng.choice(n, 64, replace=False)))
        off += n
    raw = {k: np.concatenate([r[k] for r in raws]) for k in RAWK}
    ref = np.concatenate(refs)
    outs, loss, g = T.l1_step(raw, ref, imgs, gts, 0.1, 1.0, sample=sample, fp32=True)
    rows = np.concatenate([go + sm for (H, W, s, go, gc), sm in zip(imgs, sample)])
    lay = gsr.layout([gsr.Image(H, W, s, go, gc) for (H, W, s, go, gc) in imgs])
    dev = {k: torch.from_numpy(v).cuda() for k, v in raw.items()}
    dref = torch.from_numpy(ref).cuda()
    gt_flat = torch.from_numpy(np.concatenate([x.reshape(-1) for x in gts])).cuda()
    args = (dev["raw_alpha"], dev["offset"], dref, dev["raw_sigma"], dev["raw_rho"],
            dev["raw_color"])
    direct = ops.train_step_l1(*args, lay, gt_flat, 0.1, 1.0)
    step = ops.TrainStepGraph(lay, off, ratio=0.1)
    graph = step(*args, gt_flat)
    torch.cuda.synchronize()
    cols = [("raw_alpha", [0]), ("offset", [1, 2]), ("raw_sigma", [3, 4]), ("raw_rho", [5]),
            ("raw_color", [6, 7, 8])]
    for out, gl, gg in (direct, graph):
        for k, o in enumerate(outs):
            err = np.abs(lay.view(out, k).cpu().numpy().astype(np.float64) - o)
            assert (err <= 1e-5 + 2e-6 * np.abs(o)).all(), (k, float(err.max()))
        assert float(gl.item()) == pytest.approx(loss, rel=1e-5)
        for name, c in cols:
            got = gg[name].cpu().numpy().astype(np.float64).reshape(off, -1)[rows]
            want = np.asarray(g[name]).reshape(len(rows), -1)
            S_ = g["absmass"][:, c]
            bound = (1e-4 * np.maximum(np.abs(want), 1e-1 * S_) +
                     1e-8 * S_.max(axis=0, keepdims=True))
            err = np.abs(got - want)
            assert (err <= bound + 1e-30).all(), (name, float((err / (bound + 1e-30)).max()))
