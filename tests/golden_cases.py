"""Shared helpers: load the golden fixtures written by tests/golden/make_golden.py."""

import glob
import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def case_names():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def load_case(name):
    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    arr = {k: z[k] for k in z.files}
    meta = json.loads(bytes(arr.pop("meta")).decode())
    return meta, arr
