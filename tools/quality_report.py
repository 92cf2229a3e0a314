"""Compression factor vs. relative error on the BASELINE fields (one GPU).

    python tools/quality_report.py [cfg3|cfg2|cfg1] [subdomains]

For each rank rule, reports the reference's CF accounting for
  * the fine skeleton   (sub_id layout, k (m + n) stored entries), and
  * the coarse skeleton (SPID layout, k (m_c + n), stride 2 / 3 / 4 lift),
with the exact relative Frobenius error of each reconstruction.
"""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402
from paper_2103_01380_b200.spid import RankRule  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    S = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    cfg = CONFIGS[name]
    field = CONFIGS["cfg5"] if cfg.per_gpu_subdomains else cfg
    eng = Engine(0)
    A = eng.generate(field, 0, min(S, field.subdomains))
    S, n, m = A.shape
    rows = []
    rules = [("fixed k=%d" % cfg.k, RankRule.fixed(cfg.k), cfg.k + cfg.p)]
    for kk in (2, 4, 8, 16):
        rules.append((f"fixed k={kk}", RankRule.fixed(kk), kk + cfg.p))
    for tol in (1e-3, 3e-4, 1e-4):
        rules.append((f"blocked step 2 tol {tol:g}", RankRule.blocked(64, 2, tol), 64 + cfg.p))
    for label, rule, ell in rules:
        r = eng.compress(A, ell, rule, seed=cfg.seed)
        r.check()
        e2, r2 = eng.verify(A, r)
        ks = r.rank.double()
        raw = float(m) * n * S
        row = {"rule": label, "ell": ell, "mean_rank": ks.mean().item(), "max_rank": int(ks.max()),
               "fine": {"cf": raw / (ks * (m + n)).sum().item(),
                        "rel_err": (e2.sum() / r2.sum()).sqrt().item()}}
        for stride in (2, 3, 4):
            spec = eng.block_spec(field, stride)
            mc = eng.coarse_rows(spec)
            sc = eng.gather_coarse(A, r, spec)
            ce2, cr2 = eng.verify_coarse(A, r, sc, spec)
            row[f"coarse_s{stride}"] = {"m_c": mc, "cf": raw / (ks * (mc + n)).sum().item(),
                                        "rel_err": (ce2.sum() / cr2.sum()).sqrt().item()}
        rows.append(row)
        print(json.dumps(row), flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
