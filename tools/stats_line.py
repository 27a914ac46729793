"""Compact phase-cycle line from a tools/prof_hasf.py --stats 1 JSON (stdin)."""
import json, sys
d = json.load(sys.stdin)
keys = ["ms_min", "cyc_total", "cyc_prep", "cyc_rank", "cyc_jacobi", "cyc_update", "cyc_dense", "n_dense", "cyc_dpass1",
        "cyc_dcollect", "cyc_dlist", "n_sp_big", "cyc_sp_big", "b_build", "n_build", "b_sweep", "b_rebuild",
        "n_sp_small", "cyc_sp_small", "n_tiny", "cyc_tiny", "x_tiny", "n_tinyreg", "y_top", "sweeps", "passes"]
print(" ".join(f"{k}={d[k]/1e6:.2f}M" if d.get(k, 0) > 1e5 else f"{k}={d.get(k, 0):.1f}" for k in keys))
