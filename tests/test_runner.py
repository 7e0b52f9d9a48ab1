"""Load-step runner and the SPEC output layout (paper_2209_07969_b200/runner.py).

CPU tests drive the runner through the CPU oracle (the same recipes as the B200 path); the GPU
test runs the drop-in and checks the CSV against the reference's golden table.
"""

import os

import numpy as np
import pytest

from conftest import golden
from paper_2209_07969_b200 import configs as C
from paper_2209_07969_b200 import runner as R


def _oracle():
    from oracle.phasefield_oracle import oracle_api

    return oracle_api()


def test_csv_header_only_and_round_trip(tmp_path):
    empty = R.RunReport("x", "ST")
    p = tmp_path / "e.csv"
    R.write_csv(empty, str(p))
    assert p.read_text() == "time,u,reaction,n_stag,n_nr_u,n_nr_d\n"
    rep = R.RunReport("x", "S1", [R.ReportRow(1.0, 1e-4, 12.345678901234567, 1, 2, 3),
                                  R.ReportRow(2.0, 2e-4, -0.1, 4, 5, 6),
                                  R.ReportRow(3.0, 3e-4, 1e-300, 7, 8, 9)])
    R.write_csv(rep, str(p))
    assert len(p.read_text().splitlines()) == 4
    back = R.read_csv(str(p))
    assert [(r.time, r.u, r.reaction, r.n_stag, r.n_nr_u, r.n_nr_d) for r in back] == \
        [(r.time, r.u, r.reaction, r.n_stag, r.n_nr_u, r.n_nr_d) for r in rep.rows]
    assert rep.total_n_stag == 12 and rep.max_n_stag == 7 and rep.peak_force == 12.345678901234567


def test_vtk_snapshot_layout(tmp_path):
    from types import SimpleNamespace

    mesh = SimpleNamespace(  # 2 cells, 6 nodes
        nodes=np.array([[0, 0], [1, 0], [2, 0], [0, 1], [1, 1], [2, 1]], dtype=float),
        elements=np.array([[0, 1, 4, 3], [1, 2, 5, 4]]))
    u = np.arange(12, dtype=float)
    d = np.linspace(0.0, 1.0, 6)
    p = tmp_path / "m.vtk"
    R.write_vtk_snapshot(mesh, u, d, str(p))
    lines = p.read_text().splitlines()
    assert lines[0].startswith("# vtk DataFile") and lines[2] == "ASCII"
    assert lines[3] == "DATASET UNSTRUCTURED_GRID"
    i = lines.index("POINTS 6 double")
    assert lines[i + 7] == "CELLS 2 10" and lines[i + 8].split()[0] == "4"
    j = lines.index("CELL_TYPES 2")
    assert lines[j + 1: j + 3] == ["9", "9"]
    k = lines.index("POINT_DATA 6")
    assert lines[k + 1] == "SCALARS d double 1" and lines[k + 2] == "LOOKUP_TABLE default"
    assert [float(v) for v in lines[k + 3: k + 9]] == list(d)
    v = lines.index("VECTORS u double")
    assert len(lines) - v - 1 == 6 and lines[v + 1].split() == ["0.0", "1.0", "0.0"]
    with pytest.raises(ValueError):
        R.write_vtk_snapshot(mesh, u[:4], d, str(p))


def test_config_parsing_and_errors(tmp_path):
    good = tmp_path / "ok.ini"
    good.write_text("[problem]\ncase = tension16\nscheme = S2\n[loading]\nsteps = 3\n"
                    "[output]\ndir = out\nvtk_every = 2\n")
    cfg = R.parse_config(str(good))
    assert (cfg.case, cfg.scheme, cfg.n_steps, cfg.out, cfg.vtk_every) == \
        ("tension16", "S2", 3, "out", 2)
    for text, needle in (("[problem]\ncolour = red\n", ":2: unknown key"),
                         ("[mesh]\nnx = 3\n", "unknown section"),
                         ("[loading]\nsteps = many\n", ":2: invalid value"),
                         ("[problem]\nscheme = S9\n", "unknown scheme"),
                         ("[loading]\nincrement = -1\n", "increment must be > 0")):
        bad = tmp_path / "bad.ini"
        bad.write_text(text)
        with pytest.raises(ValueError, match=needle):
            R.parse_config(str(bad))


def test_oracle_run_matches_golden_table(tmp_path):
    """The runner drives any API: through the CPU oracle the first steps of tension16 reproduce
    the reference's golden per-step counts and reactions, and the CSV is deterministic."""
    z = golden("run_tension16_S1.npz")
    tab = z["table"]
    cfg = R.RunConfig("tension16", "S1", n_steps=3, out=str(tmp_path), vtk_every=2)
    rep = R.run_benchmark(cfg, api=_oracle())
    assert [r.n_stag for r in rep.rows] == [int(x) for x in tab[:3, 1]]
    fpeak = np.abs(tab[:, 7]).max()
    assert np.allclose([r.reaction for r in rep.rows], tab[:3, 7], atol=1e-9 * fpeak)
    csv1 = (tmp_path / "tension16_S1.csv").read_bytes()
    assert sorted(os.listdir(tmp_path)) == ["tension16_S1.csv", "tension16_S1_00002.vtk",
                                            "tension16_S1_00003.vtk"]
    R.run_benchmark(cfg, api=_oracle())
    assert (tmp_path / "tension16_S1.csv").read_bytes() == csv1


@pytest.mark.gpu
def test_gpu_runner_and_sweep(cuda_ok, tmp_path):
    """The B200 drop-in through the runner: per-step counts / reactions of the golden table on
    the pre-crack steps, a sweep CSV over the four schemes."""
    z = golden("run_tension16_ST.npz")
    tab = z["table"]
    reps = R.sweep(R.RunConfig("tension16", n_steps=6, out=str(tmp_path)))
    assert [r.scheme for r in reps] == list(R.SCHEMES)
    st = reps[0]
    assert [r.n_stag for r in st.rows] == [int(x) for x in tab[:6, 1]]
    fpeak = np.abs(tab[:, 7]).max()
    assert np.allclose([r.reaction for r in st.rows], tab[:6, 7], atol=1e-6 * fpeak)
    lines = (tmp_path / "tension16_sweep.csv").read_text().splitlines()
    assert lines[0] == ",".join(R.SWEEP_HEADER) and len(lines) == 5
