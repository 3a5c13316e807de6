"""The reference's run driver (sdmortar.driver.run_config: build_from_config ->
run_method -> output.write_outputs) with this package's device run_method
swapped in -- the one-line integration INTEGRATION.md describes -- writes
byte-identical outputs on reruns and for any `workers` (the reference's own
test_driver.py:98-114 contract), for Methods S3 and S2."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN


def _cfg(name):
    from sdmortar.config import validate_config
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return validate_config(json.loads(str(z["config_json"])))


def _files(paths):
    out = [paths["moments_csv"], paths["stats_csv"], paths["manifest"]] + list(paths["vtk"])
    return {os.path.basename(p): open(p, "rb").read() for p in out}


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["S3", "S2"])
def test_device_driver_reruns_are_byte_identical(gpu, tmp_path, monkeypatch, method):
    import sdmortar.driver as drv

    from paper_1802_06263_b200 import interface
    monkeypatch.setattr(drv, "run_method", interface.run_method)
    cfg = _cfg("darcy_twoblock")
    runs = {}
    for sub, workers in (("a", 1), ("b", 1), ("w4", 4)):
        _, _, res, paths = drv.run_config(cfg, overrides={"out_dir": str(tmp_path / sub),
                                                          "method": method,
                                                          "workers": workers})
        assert isinstance(res, interface.RunResult)
        runs[sub] = _files(paths)
    assert runs["a"] == runs["b"]
    assert runs["a"] == runs["w4"]
    man = json.loads(runs["a"]["manifest.json"])
    assert "wall" not in json.dumps(man)
    # the stats rows carry the method that ran (the reference's test_method_override)
    assert runs["a"]["stats.csv"].decode().splitlines()[1].startswith(method + ",")
