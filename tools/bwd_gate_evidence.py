"""Evidence for the backward parity gate (R18 vs SURVEY 8(c).18).

For C1, C2 and C4 (sampled Gaussians), image-like and stress inputs, computes the GPU gradients
and the float64 oracle's, and reports per gradient component (alpha, mu_x, mu_y, sigma_x,
sigma_y, rho, c_r, c_g, c_b):
  * worst err / bound under SURVEY 8(c).18's gate  |g - g_ref| <= 1e-4 max(|g_ref|, 1e-2 S_t),
    S_t = sum over pairs of |term|  (oracle termabs);
  * the same with an absolute floor of 1e-8 x the largest S_t;
  * worst err / bound under the image-like test gate (tests/_util.gate_bounds, "image"):
    1e-4 max(|g|, 1e-2 S) + 1e-8 max S, S = sum of |monomials| (oracle absmass);
  * worst err / bound under R18's gate (tests/_util.gate_bounds, dist="stress");
  * err / S_t quantiles.
usage: python tools/bwd_gate_evidence.py [out.json]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import gsr_synth as S
import oracle as O
import paper_2501_06838_b200 as gsr
from _util import KEYS, flat9, gate_bounds, grad_dict, to_dev

COLS = ["alpha", "mu_x", "mu_y", "sigma_x", "sigma_y", "rho", "c_r", "c_g", "c_b"]


def summarize(got, want):
    g, w = flat9(got), flat9(want)
    err = np.abs(g - w)
    St = want["termabs"]
    survey = 1e-4 * np.maximum(np.abs(w), 1e-2 * St)
    survey_abs = survey + 1e-8 * St.max(axis=0, keepdims=True)      # + 1e-8 max S_t floor
    r18 = gate_bounds(want, want["absmass"], dist="stress")
    Sm = want["absmass"]
    mono2 = gate_bounds(want, Sm, dist="image")                      # the image-like test gate
    rs = err / np.maximum(St, 1e-300)
    out = {}
    for j, c in enumerate(COLS):
        out[c] = {"worst_ratio_survey_gate": float((err[:, j] / (survey[:, j] + 1e-30)).max()),
                  "worst_ratio_survey_gate_abs_floor": float((err[:, j] /
                                                              (survey_abs[:, j] + 1e-30)).max()),
                  "worst_ratio_r18_gate": float((err[:, j] / (r18[:, j] + 1e-30)).max()),
                  "worst_ratio_mono_1e-2_gate": float((err[:, j] / (mono2[:, j] + 1e-30)).max()),
                  "err_over_St_p50": float(np.quantile(rs[:, j], 0.5)),
                  "err_over_St_p99": float(np.quantile(rs[:, j], 0.99)),
                  "err_over_St_max": float(rs[:, j].max())}
    out["all"] = {"worst_ratio_survey_gate": max(v["worst_ratio_survey_gate"] for v in out.values()),
                  "worst_ratio_survey_gate_abs_floor": max(v["worst_ratio_survey_gate_abs_floor"]
                                                           for v in out.values()),
                  "worst_ratio_r18_gate": max(v["worst_ratio_r18_gate"] for v in out.values()
                                              if isinstance(v, dict) and "err_over_St_p50" in v),
                  "worst_ratio_mono_1e-2_gate": max(v["worst_ratio_mono_1e-2_gate"]
                                                    for v in out.values()),
                  "entries": int(err.size)}
    # the worst entries under the survey gate (+ floor): value, error and both mass scales
    ratio = err / (survey_abs + 1e-30)
    worst = []
    for f in np.argsort(-ratio, axis=None)[:6]:
        i, j = np.unravel_index(f, ratio.shape)
        worst.append({"entry": [int(i), COLS[j]], "ref": float(w[i, j]), "gpu": float(g[i, j]),
                      "err": float(err[i, j]), "S_t": float(St[i, j]), "S_mono": float(Sm[i, j]),
                      "ratio_survey_abs": float(ratio[i, j])})
    out["all"]["worst_entries_survey_abs"] = worst
    return out


def single(H, W, s, seed, gseed, dist, idx_count=None):
    c = S.gaussians(H, W, seed=seed, dist=dist)
    Hs, Ws = O.out_dims(H, W, s)
    g = S.grad_out((Hs, Ws, 3), seed=gseed)
    dev = to_dev(c)
    got = grad_dict(gsr.render_bwd(*dev, H, W, s, torch.from_numpy(g).cuda()))
    idx = None
    if idx_count:
        idx = np.random.default_rng(1).choice(c["alpha"].shape[0], idx_count, replace=False)
        got = {k: v[idx] for k, v in got.items()}
    want = O.render_bwd(c, H, W, s, 0.1, g, idx=idx, want_absmass=True)
    return summarize(got, want)


def c2(dist):
    imgs = [(48, 48, float(s)) for s in S.c2_scales()]
    res = []
    for k, (H, W, s) in enumerate(imgs):
        res.append(single(H, W, s, 1002 + 17 * k, 2002 + k, dist))
    tot = {}
    for c in COLS + ["all"]:
        tot[c] = {key: max(r[c][key] for r in res) for key in res[0][c]
                  if key not in ("entries", "worst_entries_survey_abs")}
    tot["all"]["worst_entries_survey_abs"] = sorted(
        sum((r["all"]["worst_entries_survey_abs"] for r in res), []),
        key=lambda e: -e["ratio_survey_abs"])[:8]
    return tot


def main():
    gsr.load()
    res = {}
    for dist in ("image", "stress"):
        res[f"C1/{dist}"] = single(48, 48, 4.0, 1001, 2001, dist)
        res[f"C2/{dist}"] = c2(dist)
        res[f"C4/{dist} (300 sampled Gaussians)"] = single(45, 68, 30.0, 1004, 2004, dist, 300)
    for k, v in res.items():
        print(f"{k:40s} survey-gate worst {v['all']['worst_ratio_survey_gate']:.3f}  "
              f"survey+abs-floor worst {v['all']['worst_ratio_survey_gate_abs_floor']:.3f}  "
              f"mono-1e-2 worst {v['all']['worst_ratio_mono_1e-2_gate']:.3f}  "
              f"R18-gate worst {v['all']['worst_ratio_r18_gate']:.3f}")
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/r02_bwd_gate.json"
    Path(out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
