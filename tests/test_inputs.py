"""Generator fingerprints -- the inputs both sides read."""
import json
import math
import os

import numpy as np
import pytest

from inputs import configs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fingerprints.json")))


def _check(c, g):
    assert c.n == g["N"]
    assert (float(c.x[0]), float(c.y[0])) == tuple(g["p0"])
    assert (float(c.x[-1]), float(c.y[-1])) == tuple(g["plast"])
    dig = len(g["fsum"][0].split(".")[1])
    assert f"{math.fsum(c.x):.{dig}f}" == g["fsum"][0]
    assert f"{math.fsum(c.y):.{dig}f}" == g["fsum"][1]


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_fingerprint(k, cfg_cache):
    _check(cfg_cache(k), GOLD[str(k)])


def test_fingerprint_cfg5():
    _check(configs.config5(16_000_000, grid=16), GOLD["5"])


def test_cfg4_shape_params():
    _, dc, dr, hc, hr = configs.config4_shape()
    # dc[0], dr[0], hc[0].x, hr[0]
    assert tuple(dc[0]) == (0.1685193337148995, 0.28944840527687976)
    assert dr[0] == 0.05355599642657887
    assert hc[0][0] == 0.8011447224461763
    assert hr[0] == 0.009688882408239782


def test_grids_node_centred():
    c = configs.config1()
    assert c.phi.shape == (128, 128)
    # box SDF at corner node (0,0) is 0, centre node ~ -0.5
    assert c.phi[0, 0] == 0.0
    assert abs(c.phi[64, 64] + (0.5 - abs(64 / 127 - 0.5))) < 1e-15
    X = configs.node_coords(-1.1, 1.1, 512)
    assert X[0] == -1.1 and X[-1] == 1.1
