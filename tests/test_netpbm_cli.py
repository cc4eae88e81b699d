"""Netpbm I/O, metrics and the command line against the
reference command line's own output bytes (tests/golden/cli.npz, written by
make_golden.py running pdehaze.cli)."""

import csv
import io
import json
import os

import numpy as np
import pytest

from conftest import TAU_STABLE, load_golden


@pytest.fixture(scope="module")
def g_cli():
    return load_golden("cli.npz")


def _write(path, blob):
    with open(path, "wb") as fh:
        fh.write(np.asarray(blob, dtype=np.uint8).tobytes())
    return str(path)


# ------------------------------------------------------------------ host only

def test_load_image_matches_reference_including_comments(tmp_path, g_cli):
    from paper_2506_08793_b200 import load_image

    got = load_image(_write(tmp_path / "c.ppm", g_cli["file_commented_ppm"]))
    np.testing.assert_array_equal(got, g_cli["commented_values"])
    clean = load_image(_write(tmp_path / "clean.ppm", g_cli["file_clean_ppm"]))
    assert clean.shape == (48, 64, 3) and clean.dtype == np.float64
    gray = load_image(_write(tmp_path / "g.pgm", g_cli["file_gray_pgm"]))
    assert gray.shape == (48, 64, 1)


@pytest.mark.parametrize("blob,match", [
    (b"P3\n1 1\n255\n\x00", "not a binary Netpbm"),
    (b"P5\nx 1\n255\n\x00", "expected integer width"),
    (b"P5\n2 2\n255\n\x00", "truncated payload"),
    (b"P5\n1 1\n65535\n\x00\x00", "unsupported maxval"),
    (b"P5\n1 1", "unexpected end of header"),
    (b"P5\n0 1\n255\n", "non-positive dimensions"),
    (b"P5\n1 1\n255", "missing whitespace after maxval"),
])
def test_load_image_errors(tmp_path, blob, match):
    from paper_2506_08793_b200 import NetpbmError, load_image

    p = tmp_path / "bad.pnm"
    p.write_bytes(blob)
    with pytest.raises(NetpbmError, match=match):
        load_image(str(p))
    assert issubclass(NetpbmError, ValueError)


def test_cli_defaults_are_the_reference_settings():
    from paper_2506_08793_b200 import SolverConfig
    from paper_2506_08793_b200.cli import build_parser

    args = build_parser().parse_args(["dehaze", "a", "b"])
    cfg = SolverConfig()
    for flag, field in (("omega", "omega"), ("epsilon", "epsilon"), ("sigma", "sigma"),
                        ("kernel_size", "kernel_size"), ("lambda0", "lambda0"),
                        ("beta", "beta"), ("tau", "tau"), ("t_floor", "t_floor"),
                        ("patch_radius", "patch_radius"), ("max_iters", "max_iters"),
                        ("rel_tol", "rel_tol")):
        assert getattr(args, flag) == getattr(cfg, field), flag
    assert args.lambda_monotonicity == cfg.lambda_monotonicity


def test_cli_rejects_bad_flags_before_reading_input(tmp_path, capsys):
    from paper_2506_08793_b200.cli import main

    missing = str(tmp_path / "missing.ppm")
    assert main(["dehaze", missing, str(tmp_path / "o.ppm"), "--tau", "-1"]) == 1
    err = capsys.readouterr().err.strip().splitlines()
    assert len(err) == 1 and err[0].startswith("pdehaze: error:") and "tau" in err[0]
    assert main(["synthesize", missing, str(tmp_path / "o.ppm"), "--t", "0.5",
                 "--airlight", "1.5"]) == 1
    assert "airlight" in capsys.readouterr().err
    assert main(["dehaze", missing, str(tmp_path / "o.ppm")]) == 1  # then the input
    assert "No such file" in capsys.readouterr().err
    with pytest.raises(SystemExit):
        main(["dehaze", missing, str(tmp_path / "o.ppm"), "--ablate", "no-such-stage"])
    with pytest.raises(SystemExit):
        main(["synthesize", missing, str(tmp_path / "o.ppm"), "--airlight", "0.5"])
    assert not os.path.exists(tmp_path / "o.ppm")


# ------------------------------------------------------------------ GPU

def _bytes(path):
    with open(path, "rb") as fh:
        return np.frombuffer(fh.read(), dtype=np.uint8)


@pytest.mark.gpu
def test_cli_synthesize_is_byte_exact(tmp_path, g_cli):
    from paper_2506_08793_b200.cli import main

    clean = _write(tmp_path / "clean.ppm", g_cli["file_clean_ppm"])
    tmap = _write(tmp_path / "tmap.pgm", g_cli["file_tmap_pgm"])
    assert main(["synthesize", clean, str(tmp_path / "h.ppm"), "--t", "0.4",
                 "--airlight", "0.8,0.85,0.9"]) == 0
    np.testing.assert_array_equal(_bytes(tmp_path / "h.ppm"), g_cli["file_hazy_ppm"])
    assert main(["synthesize", clean, str(tmp_path / "hm.ppm"), "--t-map", tmap,
                 "--airlight", "0.9"]) == 0
    np.testing.assert_array_equal(_bytes(tmp_path / "hm.ppm"), g_cli["file_hazy_map_ppm"])


@pytest.mark.gpu
def test_cli_dehaze_matches_the_reference_files(tmp_path, g_cli):
    from paper_2506_08793_b200.cli import main

    hazy = _write(tmp_path / "hazy.ppm", g_cli["file_hazy_ppm"])
    # no-pde: clamped inversion of the bit-exact front end -> identical bytes
    assert main(["dehaze", hazy, str(tmp_path / "n.ppm"), "--tau", repr(TAU_STABLE),
                 "--ablate", "no-pde"]) == 0
    np.testing.assert_array_equal(_bytes(tmp_path / "n.ppm"), g_cli["file_nopde_ppm"])
    # full default pipeline (multiscale + guided), 30 stable sweeps: the float32
    # solve is within 1e-4 of the float64 reference, so a sample may land one
    # quantisation step away only when it sits on a rounding boundary
    trace = str(tmp_path / "trace.csv")
    assert main(["dehaze", hazy, str(tmp_path / "d.ppm"), "--tau", repr(TAU_STABLE),
                 "--max-iters", "30", "--rel-tol", "1e-300", "--trace", trace]) == 0
    ours, ref = _bytes(tmp_path / "d.ppm").astype(int), g_cli["file_dehazed_ppm"].astype(int)
    assert ours.shape == ref.shape
    assert np.abs(ours - ref).max() <= 1 and np.count_nonzero(ours != ref) <= 8
    rows = list(csv.reader(open(trace)))
    ref_rows = list(csv.reader(io.StringIO(str(g_cli["trace_csv"]))))
    assert rows[0] == ref_rows[0] == ["channel", "iteration", "residual_norm"]
    assert [r[:2] for r in rows] == [r[:2] for r in ref_rows]
    np.testing.assert_allclose([float(r[2]) for r in rows[1:]],
                               [float(r[2]) for r in ref_rows[1:]], rtol=1e-5)
    # grayscale P5 through the same command
    gray = _write(tmp_path / "g.pgm", g_cli["file_gray_pgm"])
    assert main(["dehaze", gray, str(tmp_path / "go.pgm"), "--tau", repr(TAU_STABLE),
                 "--max-iters", "20", "--rel-tol", "1e-300", "--ablate", "no-guided"]) == 0
    ours = _bytes(tmp_path / "go.pgm").astype(int)
    ref = g_cli["file_gray_out_pgm"].astype(int)
    assert np.abs(ours - ref).max() <= 1 and np.count_nonzero(ours != ref) <= 4


@pytest.mark.gpu
def test_cli_dehaze_is_deterministic_across_runs_and_workers(tmp_path, g_cli):
    from paper_2506_08793_b200.cli import main

    hazy = _write(tmp_path / "hazy.ppm", g_cli["file_hazy_ppm"])
    blobs = []
    for name, workers in (("a", "1"), ("b", "1"), ("c", "4")):
        out = str(tmp_path / f"{name}.ppm")
        assert main(["dehaze", hazy, out, "--workers", workers, "--max-iters", "15"]) == 0
        blobs.append(_bytes(out).tobytes())
    assert blobs[0] == blobs[1] == blobs[2]


@pytest.mark.gpu
def test_cli_evaluate_matches_reference_json(tmp_path, g_cli, capsys):
    from paper_2506_08793_b200.cli import main

    clean = _write(tmp_path / "c.ppm", g_cli["file_clean_ppm"])
    hazy = _write(tmp_path / "h.ppm", g_cli["file_hazy_ppm"])
    assert main(["evaluate", clean, hazy]) == 0
    got = json.loads(capsys.readouterr().out)
    ref = json.loads(str(g_cli["evaluate_json"]))
    assert set(got) == {"mse", "psnr", "mae"}
    for k in got:
        assert got[k] == pytest.approx(ref[k], rel=1e-12)
    assert main(["evaluate", clean, clean]) == 0
    assert json.loads(capsys.readouterr().out)["psnr"] == "inf"


@pytest.mark.gpu
def test_save_image_quantisation(tmp_path):
    from paper_2506_08793_b200 import load_image, save_image

    v = np.array([[[0.0, 0.5 / 255, 1.5 / 255], [-0.2, 1.2, 254.5 / 255]]])
    save_image(v, str(tmp_path / "q.ppm"))
    raw = (tmp_path / "q.ppm").read_bytes()
    assert raw.startswith(b"P6\n2 1\n255\n")
    np.testing.assert_array_equal(np.frombuffer(raw[-6:], np.uint8), [0, 1, 2, 0, 255, 255])
    rng = np.random.default_rng(3)
    q = rng.integers(0, 256, size=(9, 11, 3)) / 255.0
    save_image(q, str(tmp_path / "r.ppm"))
    np.testing.assert_array_equal(load_image(str(tmp_path / "r.ppm")), q)
    save_image(q[:, :, 0], str(tmp_path / "g.pgm"))
    assert (tmp_path / "g.pgm").read_bytes().startswith(b"P5\n11 9\n255\n")
    with pytest.raises(ValueError):
        save_image(np.full((2, 2, 3), np.nan), str(tmp_path / "bad.ppm"))
