"""locality_metric (bench.py:236-260) against the reference's value on
tests/golden/bench.npz (host kNN over means, like the reference)."""

import pytest

from conftest import golden
from paper_2509_07782_b200.analysis import locality_metric, pipeline_config
from paper_2509_07782_b200.config import RenderConfig


def test_locality_metric_matches_reference():
    g = golden("bench")
    assert locality_metric(g["loc.means"]) == float(g["loc.identity"])
    assert locality_metric(g["loc.means"], g["loc.perm"]) == float(g["loc.morton"])
    assert locality_metric(g["loc.means"][:1]) == 0.0


def test_pipeline_config():
    base = RenderConfig()
    assert pipeline_config("uniform", base).ess is False
    assert pipeline_config("ess+adaptive", base).mode == "adaptive"
    with pytest.raises(ValueError):
        pipeline_config("bogus", base)
