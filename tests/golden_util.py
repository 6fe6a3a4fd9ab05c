"""Loading the golden fixtures (tests/golden/*.npz, made by make_golden.py
from the unmodified reference) and replaying them through an engine."""
import glob
import json
import os

import numpy as np

from paper_2210_09887_b200.network import spec_from_json

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_files():
    return sorted(glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def load(path):
    z = np.load(path)
    spec = spec_from_json(json.loads(str(z["net"])))
    cfg = json.loads(str(z["cfg"]))
    return z, spec, cfg


def replay(z, engine, check_frame, check_final=None):
    """Run every golden frame through `engine`, calling
    check_frame(k, info, out, expected_info, expected_out, expected_mask, expected_ledger)."""
    frames, hs = z["frames"], z["homographies"]
    rois = z["rois"] if "rois" in z.files else None
    for k in range(len(frames)):
        info, out = engine.run_frame(frames[k], hs[k], None if rois is None else rois[k])
        check_frame(k, info, out, json.loads(str(z[f"f{k}_info"])), z[f"f{k}_out"], z[f"f{k}_mask"],
                    z[f"f{k}_ledger"])
