"""Per-rank core bytes of the sharded apply under different ownership maps.

Builds a config on one GPU, reads every middle pair's core shape, and reports,
for world = 2, 4, 8, the heaviest rank's core bytes over the mean for
(a) round-robin ownership (s % world) and (b) the byte-balanced map of
`sharded.balanced_owners` (longest-processing-time bin packing of the per-s
core bytes).  The core stage is HBM-bound, so this ratio is the phase-1
imbalance.  Usage: python tools/shard_balance.py [config ...]
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2411_03029_b200 as tb  # noqa: E402
from paper_2411_03029_b200 import _lib, configs, sharded  # noqa: E402


def pair_shapes(bf):
    d, n, L, Lc, nmid, ns, nsk, nip, nco, npm = (int(x) for x in bf.info())
    cr = np.zeros(nmid * nmid, np.int64)
    cc = np.zeros(nmid * nmid, np.int64)
    P = _lib.ptr
    _lib.check(_lib.load().oiobf_tbf_export(bf.handle, None, None, None, None, None, None, None, P(cr), P(cc), None))
    return nmid, cr.reshape(nmid, nmid), cc.reshape(nmid, nmid)  # [s, t]


def main():
    names = sys.argv[1:] or ["green_cubes_n64", "green_cubes_n256"]
    for name in names:
        cfg = configs.BY_NAME[name]
        bf = tb.tbf_construct(cfg.spec, cfg.L, cfg.tol, seed=cfg.seed)
        nmid, cr, cc = pair_shapes(bf)
        per_s = (cr * cc).sum(axis=1) * 16  # core bytes read by the owner of s
        per_t = cr.sum(axis=0) * 16         # G_{t,s} rows received by the owner of t
        rec = {"config": name, "nmid": nmid, "core_bytes": int(per_s.sum()),
               "per_s_min": int(per_s.min()), "per_s_max": int(per_s.max())}
        for W in (2, 4, 8):
            if W > nmid:
                continue
            rr = np.arange(nmid) % W
            bal = sharded.balanced_owners(per_s, W)
            for tag, own in (("round_robin", rr), ("balanced", bal)):
                loads = np.bincount(own, weights=per_s, minlength=W)
                rec[f"w{W}_{tag}_max_over_mean"] = round(float(loads.max() / loads.mean()), 4)
            balt = sharded.balanced_owners(per_t, W)
            for tag, own in (("round_robin", rr), ("balanced", balt)):
                loads = np.bincount(own, weights=per_t, minlength=W)
                rec[f"w{W}_t_{tag}_max_over_mean"] = round(float(loads.max() / loads.mean()), 4)
        print(json.dumps(rec), flush=True)
        del bf


if __name__ == "__main__":
    main()
