"""SHA-256 of every host table DevicePlan uploads (plan.HostTables.arrays()).

The fixture tests/golden/host_tables_sha.json was written by this script in
round 2 BEFORE the package's round-1 host-setup modules were deleted, i.e.
from tables built on the package's own problem/grid objects; the CPU test
tests/test_adapter.py rebuilds the tables from the reference's own objects
(sdmortar.config.build_from_config) and requires the same hashes: the
drop-in on sdmortar objects uploads byte-identical tables.

usage: python tools/host_table_hashes.py [--out FILE] [names...]
"""
import argparse
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "case1_mini", "darcy_twoblock"]


def raw_config(name):
    """configs/<name>.json, or the parsed config stored in the golden fixture."""
    if name.startswith("cfg"):
        with open(os.path.join(ROOT, "configs", name + ".json")) as fh:
            return json.load(fh)
    z = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
    return json.loads(str(z["config_json"]))


def table_hashes(problem, grid):
    from paper_1802_06263_b200.plan import HostTables
    arrs = HostTables(problem, grid).arrays()
    return {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()[:32]
            + f":{v.dtype.str}:{'x'.join(map(str, v.shape))}"
            for k, v in sorted(arrs.items())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "host_tables_sha.json"))
    ap.add_argument("names", nargs="*")
    a = ap.parse_args()
    from paper_1802_06263_b200._ref import sdmortar  # noqa: F401
    from sdmortar.config import build_from_config, validate_config
    out = {}
    for name in a.names or NAMES:
        raw = raw_config(name)
        problem, grid, _ = build_from_config(validate_config(raw))
        out[name] = table_hashes(problem, grid)
        print(name, len(out[name]), "tables", flush=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
        fh.write("\n")


if __name__ == "__main__":
    main()
