"""Result bundle of a load program: layouts of
proj/README.md "Result bundle", io.cpp write/read round trip, averages.csv
reproduced bitwise by reloading and re-averaging."""
import csv
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hb():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2203_02962_b200 as mod
    return mod


@pytest.mark.parametrize("thermal", [False, True])
def test_result_bundle_round_trip(hb, tmp_path, thermal):
    from paper_2203_02962_b200 import bundle
    g = hb.Grid((12, 10), (1.0, 1.0), "two-triangles")
    ph = np.zeros(120, np.uint8)
    ph.reshape(12, 10)[3:8, 2:6] = 1
    if thermal:
        mats = [hb.Material.isotropic_conductivity(1.0, 2), hb.Material.isotropic_conductivity(10.0, 2)]
        loads = [[1.0, 0.0], [0.0, 1.0]]
    else:
        mats = [hb.Material.isotropic_elastic(1.0, 0.5, 2), hb.Material.j2_plastic(2.0, 1.0, 2e-3, 0.05, 2)]
        loads = [[2e-3, -1e-3, 2e-3], [4e-3, -2e-3, 4e-3]]
    res = hb.run_load_program(g, mats, ph, loads, eta_cg=1e-10, eta_newton=1e-8)
    out = str(tmp_path / "bundle")
    bundle.write_result_bundle(out, g, ph, thermal, res, seed=7)
    names = sorted(os.listdir(out))
    dual, primal = ("flux", "gradient") if thermal else ("stress", "strain")
    for i in range(2):
        for stem in (f"u_step{i}", f"{primal}_step{i}", f"{dual}_step{i}"):
            assert stem + ".f64" in names and stem + ".meta.json" in names
    u0, meta = bundle.read_field(os.path.join(out, "u_step0"))
    assert meta["layout"] == "node-planar" and list(u0.shape) == [1 if thermal else 2, g.num_nodes]
    assert np.array_equal(u0, res[0]["u"])
    rows = list(csv.reader(open(os.path.join(out, "averages.csv"))))
    m = 2 if thermal else 3
    assert rows[0][0] == "step" and len(rows) == 3
    for i in range(2):
        s, _ = bundle.read_field(os.path.join(out, f"{dual}_step{i}"))
        again = bundle._volume_average(g, s)
        assert [float(v) for v in rows[1 + i][1 + m:]] == list(again)  # bitwise
        np.testing.assert_allclose(again, res[i]["average_stress"], rtol=1e-12, atol=1e-15)
        eps, _ = bundle.read_field(os.path.join(out, f"{primal}_step{i}"))
        np.testing.assert_allclose(bundle._volume_average(g, eps), loads[i], atol=1e-12)
    rep = list(csv.reader(open(os.path.join(out, "report.csv"))))
    assert rep[0] == ["load_step", "newton_step", "cg_iterations", "residual_initial", "residual_final",
                      "increment_rel", "precond_reassembled"]
    assert json.load(open(os.path.join(out, "solve.json")))["seed"] == 7
    assert np.array_equal(np.fromfile(os.path.join(out, "phases.u8"), dtype=np.uint8), ph)
