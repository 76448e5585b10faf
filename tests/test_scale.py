"""Scale study (reference scale.py): validation and sampling on the
CPU; device gaps vs golden studies recorded from the reference (bit-exact),
the reference's c8 acceptance case and CLI cases on the GPU."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2605_19945_b200 as gem
from paper_2605_19945_b200.errors import ValidationError

GOLDEN = Path(__file__).resolve().parent / "golden" / "scale_vectors.json"


@pytest.mark.parametrize("kind,params", [("uniform", (0.0, 1.0)), ("uniform", (1.2, 1.1)), ("normal", (0.0, 1.0)),
                                         ("normal", (1.0, -0.1)), ("two_point", (1.0, 1.5, 0.9)),
                                         ("two_point", (1.0, 0.5)), ("empirical", ()), ("empirical", (1.0, -2.0)),
                                         ("poisson", (1.0,))])
def test_distribution_validation(kind, params):
    with pytest.raises(ValidationError):
        gem.ThroughputDistribution(kind, params)


def test_study_argument_validation():
    d = gem.ThroughputDistribution.uniform(0.9, 1.1)
    for sizes, samples in (((), 10), ((0, 2), 10), ((2, 2), 10), ((4, 2), 10), ((1, 2), 0)):
        with pytest.raises(ValidationError):
            gem.run_study(d, sizes, samples, 0)


def test_sampling_matches_reference_calls():
    """Same generator, same calls: the draws are the reference's (scale.py:67-76)."""
    rng_a, rng_b = np.random.default_rng(3), np.random.default_rng(3)
    d = gem.ThroughputDistribution.normal(0.02, 1.0)
    got = d.sample(rng_a, (50, 7))
    want = np.maximum(rng_b.normal(0.02, 1.0, (50, 7)), 1e-12)
    assert np.array_equal(got, want) and got.min() == 1e-12
    e = gem.ThroughputDistribution.empirical([0.9, 1.0])
    assert np.array_equal(e.sample(np.random.default_rng(1), (4, 4)),
                          np.random.default_rng(1).choice(np.asarray([0.9, 1.0]), size=(4, 4)))


@pytest.mark.gpu
def test_run_study_matches_reference_goldens():
    for case in json.loads(GOLDEN.read_text()):
        r = gem.run_study(gem.ThroughputDistribution(case["kind"], case["params"]), case["sizes"], case["samples"],
                          case["seed"])
        assert [float(g).hex() for g in r.expected_gap] == case["expected_gap"], case["kind"]
        assert r.sizes == tuple(case["sizes"]) and r.num_samples == case["samples"] and r.rng_seed == case["seed"]


@pytest.mark.gpu
def test_c8_scale_study():
    """pkg/tests/test_acceptance.py:295-309."""
    dist = gem.ThroughputDistribution.two_point(1.0, 0.5, 0.9)
    exact = (1.0 - 0.5 ** 2 - 0.5 ** 2) * (1.0 - 0.9) / 1.0
    assert abs(gem.expected_gap(dist, 2, 100_000, seed=8) - exact) <= 0.005
    study = gem.run_study(dist, (1, 2, 4, 8, 16, 32, 64), 50_000, seed=8)
    assert study.expected_gap[0] == 0.0
    assert list(study.expected_gap) == sorted(study.expected_gap)


@pytest.mark.gpu
def test_cli_scale_study(tmp_path, capsys):
    """pkg/tests/test_cli.py:158-178."""
    from paper_2605_19945_b200 import cli

    out, csv_out = tmp_path / "s.json", tmp_path / "s.csv"
    assert cli.main(["scale-study", "--dist", "two_point", "--params", "1.0,0.5,0.9", "--sizes", "1,2,4",
                     "--samples", "20000", "--seed", "2", "--output", str(out), "--csv-out", str(csv_out),
                     "--quiet"]) == 0
    payload = json.loads(out.read_text())
    gaps = payload["result"]["expected_gap"]
    assert gaps[0] == 0.0 and gaps == sorted(gaps)
    want = [c for c in json.loads(GOLDEN.read_text()) if c["kind"] == "two_point"][0]
    assert [float(g).hex() for g in gaps] == want["expected_gap"]
    lines = csv_out.read_text().strip().splitlines()
    assert lines[0] == "n,expected_gap" and len(lines) == 4
    assert cli.main(["scale-study", "--dist", "uniform", "--params", "0.88,1.11", "--sizes", "1", "--samples", "100",
                     "--seed", "1", "--quiet"]) == 0
    assert json.loads(capsys.readouterr().out)["result"]["expected_gap"] == [0.0]
