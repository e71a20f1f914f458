"""lvn_cli: the reference CLI (tools/louvain_cli.cpp) over the device engine.
Mirrors cli_tests.cpp: report schema and values, membership file vs reported
modularity, zero pass budget, --report, LOUVAIN_THREADS, bench rows, convert
round trips, loader errors and exit codes (1 parse, 2 degenerate)."""

import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2501_19004_b200", "lib", "lvn_cli")
BARBELL = "0 1\n1 2\n0 2\n3 4\n4 5\n3 5\n2 3\n"

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="lvn_cli not built")


def run(args, env=None, **kw):
    e = dict(os.environ)
    e.pop("LOUVAIN_THREADS", None)
    e.update(env or {})
    return subprocess.run([CLI] + args, capture_output=True, text=True, env=e, timeout=300, **kw)


def report(text):
    scalars, rows = {}, []
    for line in text.splitlines():
        if line.startswith("row="):
            rows.append(dict(kv.split("=", 1) for kv in line.split()))
        elif "=" in line:
            k, v = line.split("=", 1)
            scalars[k] = v
    return scalars, rows


@pytest.fixture
def barbell(tmp_path):
    p = tmp_path / "barbell.tsv"
    p.write_text(BARBELL)
    return p


# ---------------------------------------------------------------- no GPU needed
def test_convert_round_trip(tmp_path, barbell):
    mtx = tmp_path / "b.mtx"
    assert run(["convert", "--input", str(barbell), "--output", str(mtx)]).returncode == 0
    lines = mtx.read_text().splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real general" and lines[1] == "6 6 7"
    assert lines[2] == "1 2 1"
    back = tmp_path / "c.tsv"
    assert run(["convert", "--input", str(mtx), "--output", str(back)]).returncode == 0
    body = [l for l in back.read_text().splitlines() if not l.startswith("#")]
    assert body == [l.replace(" ", "\t") + "\t1" for l in BARBELL.strip().splitlines()]


@pytest.mark.parametrize("text,needle", [
    ("0 1 -2\n", "negative edge weight"),
    ("0 x\n", "expected an unsigned integer"),
    ("0 1 2 3\n", "line must be"),
])
def test_tsv_parse_errors(tmp_path, text, needle):
    p = tmp_path / "bad.tsv"
    p.write_text(text)
    r = run(["detect", "--input", str(p)])
    assert r.returncode == 1 and needle in r.stderr and "line 1" in r.stderr


@pytest.mark.parametrize("text,needle", [
    ("%%MatrixMarket matrix array real general\n2 2 1\n1 1 1\n", "only coordinate"),
    ("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n", "square"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", "out of declared bounds"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1\n", "unexpected end of file"),
    ("not a banner\n", "banner"),
])
def test_mtx_parse_errors(tmp_path, text, needle):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    r = run(["detect", "--input", str(p)])
    assert r.returncode == 1 and needle in r.stderr


def test_usage_errors(barbell):
    assert run([]).returncode == 1
    assert run(["frobnicate", "--input", str(barbell)]).returncode == 1
    assert run(["detect"]).returncode == 1
    assert run(["detect", "--input", str(barbell), "--engine", "mc"]).returncode == 1
    assert run(["detect", "--input", str(barbell), "--probing", "cubic"]).returncode == 1
    assert run(["detect", "--input", "/nonexistent.tsv"]).returncode == 1


# ---------------------------------------------------------------- on the B200
gpu = pytest.mark.gpu


def needs_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a B200")


@gpu
def test_detect_report_schema(barbell):
    needs_gpu()
    r = run(["detect", "--input", str(barbell)])
    assert r.returncode == 0, r.stderr
    s, _ = report(r.stdout)
    for k in ("input", "vertices", "edges", "avg_degree", "engine", "threads", "max_passes", "max_iterations",
              "tolerance", "tolerance_drop", "aggregation_tolerance", "modularity", "communities", "passes",
              "iterations_per_pass", "phase_local_moving", "phase_aggregation", "phase_other", "pass_split",
              "wall_time", "edges_per_second", "pl_period", "probing", "value_bits"):
        assert k in s, k
    assert float(s["vertices"]) == 6 and float(s["edges"]) == 7
    assert float(s["avg_degree"]) == pytest.approx(14 / 6)
    assert s["engine"] == "gpu"
    assert float(s["modularity"]) == pytest.approx(5 / 14, abs=1e-9)
    assert int(s["communities"]) == 2
    split = float(s["phase_local_moving"]) + float(s["phase_aggregation"]) + float(s["phase_other"])
    assert split == pytest.approx(1.0, abs=1e-9)
    assert float(s["edges_per_second"]) == pytest.approx(7 / float(s["wall_time"]), rel=1e-6)


@gpu
def test_detect_membership_file(tmp_path, barbell):
    needs_gpu()
    out = tmp_path / "m.tsv"
    r = run(["detect", "--input", str(barbell), "--output", str(out)])
    assert r.returncode == 0, r.stderr
    s, _ = report(r.stdout)
    rows = [tuple(map(int, l.split())) for l in out.read_text().splitlines()]
    assert [v for v, _ in rows] == list(range(6))
    memb = [c for _, c in rows]
    assert sorted(set(memb)) == list(range(int(s["communities"])))
    assert memb[0] == memb[1] == memb[2] != memb[3] == memb[4] == memb[5]


@gpu
def test_detect_zero_passes_and_report_file(tmp_path, barbell):
    needs_gpu()
    r = run(["detect", "--input", str(barbell), "--max-passes", "0"])
    s, _ = report(r.stdout)
    assert r.returncode == 0 and int(s["communities"]) == 6 and int(s["passes"]) == 0
    rp = tmp_path / "r.txt"
    r = run(["detect", "--input", str(barbell), "--report", str(rp), "--value-bits", "64", "--probing", "double"])
    assert r.returncode == 0 and r.stdout == ""
    s, _ = report(rp.read_text())
    assert int(s["communities"]) == 2 and s["value_bits"] == "64" and s["probing"] == "double"


@gpu
def test_threads_env(barbell):
    needs_gpu()
    s, _ = report(run(["detect", "--input", str(barbell)], env={"LOUVAIN_THREADS": "3"}).stdout)
    assert s["threads"] == "3"
    s, _ = report(run(["detect", "--input", str(barbell), "--threads", "2"], env={"LOUVAIN_THREADS": "3"}).stdout)
    assert s["threads"] == "2"


@gpu
def test_bench_rows(barbell):
    needs_gpu()
    r = run(["bench", "--input", str(barbell), "--threads", "1,2", "--repetitions", "3"])
    assert r.returncode == 0, r.stderr
    s, rows = report(r.stdout)
    assert int(s["repetitions"]) == 3
    runs = [x for x in rows if x["row"] == "run"]
    scaling = [x for x in rows if x["row"] == "scaling"]
    assert len(runs) == 6 and len(scaling) == 2
    for x in runs:
        assert float(x["modularity"]) == pytest.approx(5 / 14, abs=1e-9)
    one = [x for x in scaling if x["threads"] == "1"][0]
    assert float(one["speedup"]) == pytest.approx(1.0)


@gpu
def test_degenerate_and_symmetrize(tmp_path):
    needs_gpu()
    p = tmp_path / "zero.tsv"
    p.write_text("0 1 0\n")
    assert run(["detect", "--input", str(p)]).returncode == 2
    q = tmp_path / "dup.tsv"
    q.write_text("0 1 1.5\n1 0 0.25\n2 2 3\n")
    out = tmp_path / "sym.tsv"
    assert run(["convert", "--input", str(q), "--output", str(out), "--symmetrize"]).returncode == 0
    body = [l.split("\t") for l in out.read_text().splitlines() if not l.startswith("#")]
    assert body == [["0", "1", "1.75"], ["1", "0", "1.75"], ["2", "2", "3"]]
