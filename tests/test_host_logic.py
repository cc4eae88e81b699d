"""Host-side logic that needs no GPU: configuration, ablation flags, trace
CSV, the synthetic workload generator, bench plumbing."""

import csv
import hashlib

import numpy as np
import pytest

from paper_2506_08793_b200.config import (ABLATIONS, SolverConfig, SolverTrace,
                                          normalize_ablation)


@pytest.mark.parametrize("kwargs", [
    {"epsilon": 0.0}, {"sigma": -1.0}, {"kernel_size": 4}, {"kernel_size": 0},
    {"lambda0": 0.0}, {"beta": -0.5}, {"tau": 0.0}, {"t_floor": 0.0}, {"omega": 0.0},
    {"omega": 1.5}, {"patch_radius": -1}, {"max_iters": 0}, {"rel_tol": 0.0},
    {"lambda_monotonicity": "upside-down"}, {"guided_radius": 0}, {"guided_reg": 0.0},
    {"multiscale_radii": ()}, {"airlight_fraction": 0.0},
])
def test_bad_config_rejected(kwargs):
    # the reference's TestConfigValidation cases (tests/test_solver.py:544-570)
    with pytest.raises(ValueError):
        SolverConfig(**kwargs)


def test_config_defaults():
    cfg = SolverConfig()
    assert (cfg.omega, cfg.epsilon, cfg.sigma, cfg.kernel_size, cfg.lambda0, cfg.beta,
            cfg.tau, cfg.patch_radius, cfg.t_floor, cfg.max_iters, cfg.rel_tol) == \
        (0.95, 1e-3, 2.0, 5, 0.5, 3.0, 0.2, 7, 0.1, 200, 1e-4)
    assert cfg.multiscale_radii == (3, 7, 15) and cfg.airlight_fraction == 0.001


def test_ablation_normalisation():
    assert normalize_ablation(None) == frozenset()
    assert normalize_ablation("no-pde") == frozenset({"no-pde"})
    assert normalize_ablation(["no-guided", "no-multiscale"]) == \
        frozenset({"no-guided", "no-multiscale"})
    with pytest.raises(ValueError, match="unknown ablation"):
        normalize_ablation("no-such-stage")
    assert len(ABLATIONS) == 6


def test_trace_csv(tmp_path):
    from paper_2506_08793_b200.solver import write_trace_csv

    traces = [SolverTrace(residual_norms=[1.5, 0.1 + 0.2], iterations_run=2),
              SolverTrace(residual_norms=[3.0], iterations_run=1)]
    p = tmp_path / "t.csv"
    write_trace_csv(traces, p)
    rows = list(csv.reader(open(p, newline="")))
    assert rows[0] == ["channel", "iteration", "residual_norm"]
    assert rows[1:] == [["0", "1", "1.5"], ["0", "2", repr(0.1 + 0.2)], ["1", "1", "3.0"]]


def test_synthetic_generator_deterministic():
    from paper_2506_08793_b200.synthetic import BENCH_CONFIGS, make_hazy_scene

    a = make_hazy_scene(64, 96, 2, 5)
    b = make_hazy_scene(64, 96, 2, 5)
    assert a.hazy.dtype == np.float32 and a.hazy.shape == (64, 96, 3)
    np.testing.assert_array_equal(a.hazy, b.hazy)
    assert 0.0 <= a.hazy.min() and a.hazy.max() <= 1.0
    assert 0.6 <= a.beta <= 1.6 and np.all((0.8 <= a.airlight) & (a.airlight <= 1.0))
    c = make_hazy_scene(64, 96, 2, 6)
    assert not np.array_equal(a.hazy, c.hazy)
    assert BENCH_CONFIGS[2]["kernel_size"] == 19 and BENCH_CONFIGS[2]["max_iters"] == 200


def test_config1_input_pinned(g_c1):
    from paper_2506_08793_b200.synthetic import make_hazy_scene

    s = make_hazy_scene(256, 256, 1, 0)
    assert hashlib.sha256(s.hazy.tobytes()).hexdigest() == str(g_c1["input_sha"])


def test_oracle_not_imported_by_product():
    """The product package must never import the oracle (test infrastructure)."""
    import os

    from conftest import REPO

    pkg = os.path.join(REPO, "paper_2506_08793_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                text = open(os.path.join(root, f)).read()
                for needle in ("import oracle", "from oracle", "pdz_oracle"):
                    assert needle not in text, (f, needle)


def test_bench_workloads_and_shards():
    """bench.py host logic: the `config` object is the same in both arms, the
    image shards of config 3 cover the batch exactly once for every world
    size, and the CPU arm's bounded sample is a crop of the config."""
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location(
        "bench", os.path.join(os.path.dirname(os.path.dirname(__file__)), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for n in (1, 2, 3, 4, 5):
        w = bench._workload(n)
        assert w == bench._workload(n) and w["config_number"] == n
        assert set(w) >= {"workload", "height", "width", "kernel_size", "iterations", "l2"}
        rows, cols = bench.cpu_sample_shape(n)
        assert 1 <= rows <= w["height"] and 1 <= cols <= w["width"]
        assert rows * cols * w["kernel_size"] ** 2 <= 2.1 * 1024 * 1024 * 19 * 19
    assert bench._workload(5)["rel_tol"] == 1e-5 and bench._workload(2)["rel_tol"] is None
    for world in (1, 2, 3, 4, 8):
        seen = [i for r in range(world) for i in bench.shard(256, world, r)]
        assert seen == list(range(256))
        assert max(len(bench.shard(256, world, r)) for r in range(world)) == -(-256 // world)
    assert bench._mode(3, 8)[1] == "strong" and bench._mode(2, 8)[1] == "weak"
    assert "row slabs" in bench._mode(4, 4)[0] and "replicas" in bench._mode(4, 1)[0]
