"""Problem-file I/O (problems.py:300-395) and the CLI entry point against
files written by the unmodified reference (tests/golden/make_golden_problem_io.py).
CPU only."""

import os

import numpy as np
import pytest

import paper_1802_08126_b200 as pg
from conftest import GOLDEN

FILE = os.path.join(GOLDEN, "problem_c8_N4.txt")


def test_load_reference_file():
    d = np.load(os.path.join(GOLDEN, "problem_c8_N4.npz"))
    spec = pg.load_problem(FILE)
    np.testing.assert_array_equal(spec.grid.nodes, d["nodes"])
    np.testing.assert_array_equal(spec.load, d["load"])
    np.testing.assert_array_equal(spec.u_init, d["u_init"])
    assert spec.tau_ref == float(d["tau_ref"]) and spec.alpha == float(d["alpha"])
    np.testing.assert_array_equal(spec.mass.todense(), d["mass"])
    np.testing.assert_array_equal(spec.a_ref.todense(), d["a_ref"])
    np.testing.assert_array_equal(np.stack([a.todense() for a in spec.stiffness]), d["stiff"])
    assert spec.meta == {"space": "2d", "mesh": 8}


def test_save_is_byte_identical(tmp_path):
    """Our writer reproduces the reference's file byte for byte."""
    spec = pg.load_problem(FILE)
    out = tmp_path / "p.txt"
    pg.save_problem(spec, str(out))
    assert out.read_bytes() == open(FILE, "rb").read()


def test_bad_header(tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("not-a-problem\n")
    with pytest.raises(pg.InputError):
        pg.load_problem(str(bad))


def test_cli_rejects_non_gpu_options():
    from paper_1802_08126_b200.cli import main

    assert main(["solve", "--solver", "direct"]) == 1
    assert main(["solve", "--problem-file", "/nonexistent/file"]) == 1


@pytest.mark.gpu
def test_cli_sequential_matches_oracle(tmp_path):
    """--method sequential: the time-stepping oracle's first node per step in
    the reference's CSV format (cli.py:142-145), device exact solves."""
    import numpy as np

    import oracle as orc
    from paper_1802_08126_b200.cli import main

    out = tmp_path / "seq.csv"
    assert main(["solve", "--method", "sequential", "--space", "2d", "--h", "8", "--N", "5",
                 "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "step,node" and len(lines) == 6
    spec = pg.make_heat_problem("2d", 8, pg.build_time_grid("uniform", 5, 1.0), data="sine")
    opb = orc.heat_problem("2d", 8, orc.time_nodes("uniform", 5, 1.0), load=spec.load,
                           u_init=spec.u_init)
    ref = orc.sequential_euler(opb)
    got = np.array([float(ln.split(",")[1]) for ln in lines[1:]])
    assert np.max(np.abs(got - ref[:, 0])) <= 1e-13 * np.max(np.abs(ref[:, 0])) + 1e-300


def test_cli_config_merge(tmp_path):
    """--config key=value defaults, command line wins (cli.py:32-43, 161-181)."""
    from paper_1802_08126_b200.cli import build_parser, merge_config, read_config

    conf = tmp_path / "c.conf"
    conf.write_text("# comment\nomega = 0.5\nmax-iter=7  # trailing\n\ntol=1e-3\n")
    entries = read_config(str(conf))
    assert entries == {"omega": "0.5", "max-iter": "7", "tol": "1e-3"}
    argv = merge_config(["--config", str(conf), "solve", "--tol", "1e-9"], entries)
    args = build_parser().parse_args(argv)
    assert args.omega == 0.5 and args.max_iter == 7 and args.tol == 1e-9
    bad = tmp_path / "bad.conf"
    bad.write_text("no equals sign here\n")
    from paper_1802_08126_b200.cli import main

    assert main(["--config", str(bad), "solve"]) == 1
    assert main(["--config", str(tmp_path / "missing.conf"), "solve"]) == 1
