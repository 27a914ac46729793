"""Small cases over every kernel flavour (512- and 256-thread hot variants,
cluster and cooperative teams, forced segmentation with constraints, host
and P4 entries, exact EDT, the stage path for r > 16), each against the
oracle -- a quick flavour smoke, and the input for compute-sanitizer
(memcheck / synccheck) where it is available (it is closed on this pool):
    python tools/sanitize_cases.py
Exits non-zero on any mismatch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1603_09337_b200 as P  # noqa: E402
from paper_1603_09337_b200 import _lib, workloads as W  # noqa: E402


def main():
    lib = _lib.load()
    rng = np.random.default_rng(3)
    bad = 0

    def check(tag, got, want):
        nonlocal bad
        if not np.array_equal(got, want):
            bad += 1
            print("MISMATCH", tag, flush=True)

    imgs = np.stack([(rng.random((96, 128)) < 0.5).astype(np.uint8) for _ in range(3)])
    check("hot512", P.hasf_batch(imgs, 3), O.hasf_batch(imgs, 3, 8))
    mz = W.config_batch("c4", 4000, 2)[:, :128, :128].copy()
    check("hot256_48", P.hasf_batch(mz, 2, P.ADJ_48), O.hasf_batch(mz, 2, 4))
    for team, cl in ((2, 1), (3, 0)):
        lib.ts_set_team_size(team)
        lib.ts_set_cluster_teams(cl)
        check(f"team{team}_cluster{cl}", P.hasf_batch(imgs[:1], 2), O.hasf_batch(imgs[:1], 2, 8))
    lib.ts_set_team_size(0)
    lib.ts_set_cluster_teams(1)
    lib.ts_set_segment_force(1)
    lib.ts_set_segment_stages(1)
    keep = (imgs & (rng.random(imgs.shape) < 0.05)).astype(np.uint8)
    check("segmented", P.hasf_batch(imgs, 3, keep=keep), O.hasf_batch(imgs, 3, 8, keep=keep))
    lib.ts_set_segment_force(0)
    lib.ts_set_segment_stages(8)
    check("host", P.hasf_batch_host(imgs, 2), O.hasf_batch(imgs, 2, 8))
    check("p4", np.unpackbits(P.hasf_p4(np.packbits(imgs, axis=2), 128, 2), axis=2), O.hasf_batch(imgs, 2, 8))
    check("edt", P.edt_squared(imgs[0]), O.edt_squared(imgs[0]))
    check("big_r", P.smooth(imgs[0][:48, :48].copy(), 17), O.hasf(imgs[0][:48, :48].copy(), 17, 8))
    fi, bi = P.topology_counts(imgs)
    print("sanitize cases done, mismatches:", bad, flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
