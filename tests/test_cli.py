"""kvprefill_b200 CLI vs the reference CLI (test_cli.cpp restated; commands.hpp).

CPU tests: every planning subcommand (sweep with engine runs disabled, search, predict, noise)
is byte-identical to the reference's own commands.hpp run through oracle/_ref on the same
config file, plus the reference's CLI behaviours (exit codes, skips, determinism).
GPU tests: verify and sweep's engine column run the B200 engine."""
import json
import os
import subprocess

import pytest

import oracle as O
from paper_2405_05329_b200 import build

CLI = build.CLI


def _cli():
    build.build()
    return CLI


def run_cli(args, cwd):
    r = subprocess.run([_cli(), *args], cwd=cwd, capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout, r.stderr


def write_config(tmp_path, doc, name="config.json"):
    p = tmp_path / name
    p.write_text(json.dumps(doc, indent=2))
    return str(p)


def fast_model():
    return {"d_model": 16, "n_heads": 4, "n_kv_heads": 2, "n_layers": 2, "seed": 5}


def csv_rows(text):
    lines = [ln for ln in text.splitlines() if ln]
    return [ln.split(",") for ln in lines[1:]]


@pytest.fixture(scope="module")
def ref():
    return O.Reference()


def ref_cli(ref, capfd, sub, cfg, C_=-1, out="", table=""):
    rc = ref.cli(sub, cfg, C_, out, table)
    cap = capfd.readouterr()
    return rc, cap.out, cap.err


# ------------------------------------------------------------- byte identity with the reference
SWEEPS = [
    {"context_lengths": [32, 64, 4096], "process_counts": [1, 2, 3, 4], "partition_source": "search"},
    {"context_lengths": [512, 1024], "process_counts": [4], "strategies": ["kvr"]},
    {"context_lengths": [2], "process_counts": [4], "strategies": ["tsp", "kvr"]},
    {"context_lengths": [4096], "process_counts": [1, 2], "strategies": ["serial", "kvr"],
     "partition_source": "search", "network": {"bandwidth": 1e18, "latency": 0.0}},
    {"context_lengths": [1000, 3000], "process_counts": [3], "partition_source": "ratios",
     "ratios": [0.5, 0.3, 0.2], "cost": {"alpha": 2e-6, "proj_coeff": 1e-6}, "format": "json"},
    {"context_lengths": [16384], "process_counts": [8], "partition_source": "search",
     "model": {"d_model": 4096, "n_heads": 32, "n_kv_heads": 32, "n_layers": 32}},
]


@pytest.mark.parametrize("i", range(len(SWEEPS)))
def test_sweep_byte_identical_to_reference(tmp_path, ref, capfd, i):
    doc = {"model": fast_model(), "equivalence_max_c": 0, **SWEEPS[i]}
    cfg = write_config(tmp_path, doc)
    mine, theirs = str(tmp_path / "mine.out"), str(tmp_path / "ref.out")
    rc, _, err = run_cli(["sweep", "--config", cfg, "--out", mine], tmp_path)
    rrc, _, rerr = ref_cli(ref, capfd, "sweep", cfg, out=theirs)
    assert rc == rrc == 0
    assert open(mine).read() == open(theirs).read()
    assert ("infeasible" in err) == ("infeasible" in rerr)


def test_search_predict_noise_byte_identical_to_reference(tmp_path, ref, capfd):
    doc = {"model": fast_model(), "context_lengths": [256, 512, 1024], "process_counts": [4]}
    cfg = write_config(tmp_path, doc)
    rc, out, _ = run_cli(["search", "--config", cfg, "--table", str(tmp_path / "mine.json")], tmp_path)
    rrc, rout, _ = ref_cli(ref, capfd, "search", cfg, table=str(tmp_path / "ref.json"))
    assert rc == rrc == 0
    assert open(tmp_path / "mine.json").read() == open(tmp_path / "ref.json").read()
    assert out.replace("mine.json", "X") == rout.replace("ref.json", "X")
    for C_ in (512, 768, 32, 5000):
        for fmt in ("csv", "json"):
            c2 = write_config(tmp_path, {**doc, "table_path": str(tmp_path / "mine.json"), "format": fmt}, "p.json")
            rc, _, _ = run_cli(["predict", str(C_), "--config", c2, "--out", str(tmp_path / "pm")], tmp_path)
            rrc, _, _ = ref_cli(ref, capfd, "predict", c2, C_, out=str(tmp_path / "pr"))
            assert rc == rrc == 0
            assert open(tmp_path / "pm").read() == open(tmp_path / "pr").read(), (C_, fmt)
    for fmt in ("csv", "json"):
        c3 = write_config(tmp_path, {**doc, "strategies": ["tsp", "kvr"], "format": fmt,
                                     "noise": {"slowdown_factor": 256.0, "trials": 7}}, "n.json")
        rc, out, _ = run_cli(["noise", "--config", c3, "--out", str(tmp_path / "nm")], tmp_path)
        rrc, rout, _ = ref_cli(ref, capfd, "noise", c3, out=str(tmp_path / "nr"))
        assert rc == rrc == 0
        assert open(tmp_path / "nm").read() == open(tmp_path / "nr").read()
        assert out == rout  # verdict lines


# ------------------------------------------------------------- test_cli.cpp, restated
def test_sweep_header_and_serial_rows(tmp_path):
    cfg = write_config(tmp_path, {"model": fast_model(), "context_lengths": [32, 64], "process_counts": [1, 2],
                                  "equivalence_max_c": 0, "out_path": str(tmp_path / "s.csv")})
    rc, out, _ = run_cli(["sweep", "--config", cfg], tmp_path)
    assert rc == 0 and "wrote" in out
    text = open(tmp_path / "s.csv").read()
    assert text.startswith("strategy,C,p,partition,ttft_sim,speedup,ttft_star,ttft_lower,dot_max,"
                           "pairs,rows,barriers,max_dev\n")
    rows = csv_rows(text)
    assert any(r[0] == "serial" for r in rows)
    for r in rows:
        assert len(r) == 13
        if r[0] == "serial":
            assert float(r[5]) == 1.0 and r[11] == "0"
        if r[0] == "tsp":
            assert r[11] == "2"


def test_sweep_superlinear_at_two_ranks_zero_comm(tmp_path):
    cfg = write_config(tmp_path, {"model": fast_model(), "strategies": ["serial", "kvr"], "context_lengths": [4096],
                                  "process_counts": [1, 2], "partition_source": "search",
                                  "network": {"bandwidth": 1e18, "latency": 0.0}, "equivalence_max_c": 0})
    rc, out, _ = run_cli(["sweep", "--config", cfg], tmp_path)
    assert rc == 0
    assert any(float(r[5]) > 2.0 for r in csv_rows(out) if r[0] == "kvr" and r[2] == "2")


def test_searched_partitions_never_lose_to_even(tmp_path):
    base = {"model": fast_model(), "strategies": ["kvr"], "context_lengths": [512, 1024], "process_counts": [4],
            "equivalence_max_c": 0}
    _, even, _ = run_cli(["sweep", "--config", write_config(tmp_path, base, "e.json")], tmp_path)
    _, srch, _ = run_cli(["sweep", "--config", write_config(tmp_path, {**base, "partition_source": "search"},
                                                            "s.json")], tmp_path)
    e, s = csv_rows(even), csv_rows(srch)
    assert len(e) == len(s) > 0
    for a, b in zip(e, s):
        assert float(b[4]) <= float(a[4]) * (1 + 1e-12)


def test_sweep_skips_infeasible_and_is_deterministic(tmp_path):
    cfg = write_config(tmp_path, {"model": fast_model(), "strategies": ["tsp", "kvr"], "context_lengths": [2],
                                  "process_counts": [4]})
    rc, out, err = run_cli(["sweep", "--config", cfg], tmp_path)
    assert rc == 0 and "infeasible" in err
    assert all(r[3] == "skipped" for r in csv_rows(out))
    cfg = write_config(tmp_path, {"model": fast_model(), "context_lengths": [64], "process_counts": [1, 2, 3],
                                  "equivalence_max_c": 0}, "d.json")
    a = run_cli(["sweep", "--config", cfg, "--out", str(tmp_path / "a.csv")], tmp_path)
    b = run_cli(["sweep", "--config", cfg, "--out", str(tmp_path / "b.csv")], tmp_path)
    assert a[0] == b[0] == 0
    assert open(tmp_path / "a.csv").read() == open(tmp_path / "b.csv").read()


def test_search_table_front_loaded_and_deterministic(tmp_path):
    cfg = write_config(tmp_path, {"model": fast_model(), "context_lengths": [256, 512, 1024], "process_counts": [4],
                                  "table_path": str(tmp_path / "ta.json")})
    rc, _, _ = run_cli(["search", "--config", cfg], tmp_path)
    assert rc == 0
    t = json.load(open(tmp_path / "ta.json"))
    assert t["p"] == 4 and len(t["entries"]) == 3
    for e in t["entries"]:
        assert abs(sum(e["ratios"]) - 1.0) <= 1e-9 and e["ratios"][0] >= e["ratios"][-1]
    assert run_cli(["search", "--config", cfg, "--table", str(tmp_path / "tb.json")], tmp_path)[0] == 0
    assert open(tmp_path / "ta.json").read() == open(tmp_path / "tb.json").read()
    bad = write_config(tmp_path, {"model": fast_model(), "context_lengths": [64], "process_counts": [2, 4],
                                  "table_path": str(tmp_path / "x.json")}, "bad.json")
    assert run_cli(["search", "--config", bad], tmp_path)[0] == 2


def test_predict_interpolates_and_clamps(tmp_path):
    cfg = write_config(tmp_path, {"model": fast_model(), "context_lengths": [256, 512, 1024], "process_counts": [4],
                                  "table_path": str(tmp_path / "t.json")})
    assert run_cli(["search", "--config", cfg], tmp_path)[0] == 0
    rc, out, _ = run_cli(["predict", "512", "--config", cfg], tmp_path)
    row = csv_rows(out)
    assert rc == 0 and len(row) == 1 and float(row[0][5]) == 0.0 and row[0][6] == "false"
    rc, out, _ = run_cli(["predict", "768", "--config", cfg], tmp_path)
    assert rc == 0 and float(csv_rows(out)[0][5]) <= 0.05
    rc, out, err = run_cli(["predict", "32", "--config", cfg], tmp_path)
    assert rc == 0 and "clamped" in err and csv_rows(out)[0][6] == "true"
    absent = write_config(tmp_path, {"model": fast_model(), "table_path": str(tmp_path / "absent.json")}, "a.json")
    assert run_cli(["predict", "128", "--config", absent], tmp_path)[0] == 2
    assert run_cli(["predict", "--config", absent], tmp_path)[0] == 2


def test_noise_unit_factor_and_verdict(tmp_path):
    base = {"model": fast_model(), "strategies": ["tsp", "kvr"], "context_lengths": [1024], "process_counts": [4]}
    cfg = write_config(tmp_path, {**base, "noise": {"slowdown_factor": 1.0, "trials": 4}})
    rc, out, _ = run_cli(["noise", "--config", cfg], tmp_path)
    rows = csv_rows(out)
    assert rc == 0 and len(rows) == 2
    assert all(float(r[7]) == 0.0 and float(r[8]) == 0.0 for r in rows)
    cfg = write_config(tmp_path, {**base, "noise": {"slowdown_factor": 256.0, "trials": 20},
                                  "out_path": str(tmp_path / "n.csv")}, "n.json")
    rc, out, _ = run_cli(["noise", "--config", cfg], tmp_path)
    assert rc == 0 and "KVR more robust" in out


def test_configuration_problems_exit_with_usage_code(tmp_path):
    (tmp_path / "broken.json").write_text('{ "model": ')
    rc, _, err = run_cli(["verify", "--config", str(tmp_path / "broken.json")], tmp_path)
    assert rc == 2 and "line" in err
    assert run_cli(["verify", "--config", write_config(tmp_path, {"model": fast_model(), "not_a_real_key": 1},
                                                       "u.json")], tmp_path)[0] == 2
    assert run_cli(["sweep", "--config", write_config(tmp_path, {"model": fast_model(), "format": "xml"},
                                                      "f.json")], tmp_path)[0] == 2
    bad_ratios = {"model": fast_model(), "strategies": ["kvr"], "context_lengths": [64], "process_counts": [2],
                  "partition_source": "ratios", "ratios": [0.5, 0.3, 0.2], "equivalence_max_c": 0}
    assert run_cli(["sweep", "--config", write_config(tmp_path, bad_ratios, "r.json")], tmp_path)[0] == 2
    assert run_cli(["definitely_not_a_subcommand"], tmp_path)[0] == 2


def test_json_output_matches_csv_content(tmp_path):
    doc = {"model": fast_model(), "context_lengths": [32], "process_counts": [2], "equivalence_max_c": 0}
    _, csv_out, _ = run_cli(["sweep", "--config", write_config(tmp_path, doc, "c.json")], tmp_path)
    _, js, _ = run_cli(["sweep", "--config", write_config(tmp_path, {**doc, "format": "json"}, "j.json")], tmp_path)
    rows = json.loads(js)
    assert isinstance(rows, list) and rows
    for r, c in zip(rows, csv_rows(csv_out)):
        assert r["C"] == 32 and r["strategy"] == c[0] and float(c[4]) == pytest.approx(r["ttft_sim"], rel=1e-9)


# ------------------------------------------------------------- engine-backed (B200)
@pytest.mark.gpu
def test_verify_default_configuration_passes(tmp_path):
    rc, out, err = run_cli(["verify"], tmp_path)
    assert rc == 0, out + err
    assert "all checks passed" in out


@pytest.mark.gpu
def test_verify_fixture_figures_summary_and_fault(tmp_path):
    cfg = write_config(tmp_path, {"model": {**fast_model(), "precision": "f32"}, "context_lengths": [16, 32],
                                  "process_counts": [1, 2], "out_path": str(tmp_path / "v.json")})
    rc, out, _ = run_cli(["verify", "--config", cfg], tmp_path)
    assert rc == 0, out
    for s in ("16/21/18", "27", "22 rows", "36 rows"):
        assert s in out
    summary = json.load(open(tmp_path / "v.json"))
    assert summary["all_passed"] is True and len(summary["checks"]) > 0
    cfg = write_config(tmp_path, {"model": fast_model(), "context_lengths": [16], "process_counts": [2],
                                  "fault": {"kind": "drop_message", "rank": 0, "layer": 0}}, "f.json")
    rc, out, _ = run_cli(["verify", "--config", cfg], tmp_path)
    assert rc == 1 and "[pass] fault injection surfaced" in out


@pytest.mark.gpu
def test_sweep_engine_columns(tmp_path):
    for prec in ("f32", "bf16"):
        cfg = write_config(tmp_path, {"model": {**fast_model(), "precision": prec}, "context_lengths": [32, 64],
                                      "process_counts": [1, 2, 3]}, f"{prec}.json")
        rc, out, err = run_cli(["sweep", "--config", cfg, "--measure"], tmp_path)
        assert rc == 0, err
        assert out.splitlines()[0].endswith(",max_dev,ttft_measured")
        for r in csv_rows(out):
            assert float(r[12]) == 0.0  # Serial == TSP == KVR bitwise on the GPU
            assert float(r[13]) > 0.0
