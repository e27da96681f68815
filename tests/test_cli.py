"""The drop-in CLI (paper_2002_03400_b200/cli.py) against the reference CLI's
contracts (tools/bfly_cli.cpp): options, log.json, the bfly.factorize.v1 CSV
row, the .bfh container."""
import json
import os

import numpy as np
import pytest

import oracle as O
from helpers import oracle_config


def test_cli_parser_and_formats(tmp_path):
    from paper_2002_03400_b200 import api, cli

    ap = cli.parser()
    o = ap.parse_args(["--eps", "1e-6", "--r0", "16", "--L", "5", "--csv", "x.csv", "factorize", "--config", "c.json"])
    assert (o.cmd, o.eps, o.r0, o.L, o.csv, o.config_sub) == ("factorize", 1e-6, 16, 5, "x.csv", "c.json")
    o = ap.parse_args(["synth", "--levels", "3", "--rank", "2"])
    assert (o.cmd, o.levels, o.rank, o.eps, o.oversample, o.seed) == ("synth", 3, 2, 1e-3, 2, 0)
    # std::setprecision(17) (bfly_cli.cpp:50-54)
    assert cli.fmt(0.1) == "0.10000000000000001" and cli.fmt(1e-6) == "9.9999999999999995e-07"
    p = str(tmp_path / "r.csv")
    cli.append_csv(p, cli.SCHEMA, cli.HEADER, ["a"])
    cli.append_csv(p, cli.SCHEMA, cli.HEADER, ["b"])
    assert open(p).read() == f"# schema: bfly.factorize.v1\n{cli.HEADER}\na\nb\n"
    lg = api.FactorizationLog([api.PhaseStat("leaf_v", 0, 18, 0.5, 1, 18)], 100, 2, False, 0.75, 0.0, 0.0)
    j = cli.log_to_json(lg)
    assert j["phases"][0] == {"name": "leaf_v", "forward_columns": 0, "transpose_columns": 18, "seconds": 0.5,
                              "rounds": 1, "probe_width": 18}
    assert (j["total_columns"], j["peak_probe_bytes"], j["rank_capped"], j["total_seconds"]) == (18, 100, False, 0.75)


@pytest.mark.gpu
def test_cli_factorize_matches_oracle(tmp_path, oracle_threads):
    from paper_2002_03400_b200 import cli

    cfgp = tmp_path / "cfg.json"
    cfgp.write_text(json.dumps({"operator": "helmholtz_circle", "n": 1024}))
    csv = tmp_path / "out.csv"
    rc = cli.main(["--out", str(tmp_path / "run"), "--csv", str(csv), "--eps", "1e-6", "--r0", "4",
                   "factorize", "--config", str(cfgp)])
    assert rc == 0
    op_o, rt, ct, cfg = oracle_config(2, 1024)
    bf_o, log_o = O.factorize(op_o, rt, ct, dict(cfg, threads=oracle_threads))
    lines = open(csv).read().splitlines()
    assert lines[0] == "# schema: bfly.factorize.v1" and lines[1] == cli.HEADER
    kind, n, L, eps, max_rank, err, secs, nbytes, cols = lines[2].split(",")
    assert (kind, int(n), int(L), float(eps)) == ("helmholtz_circle", 1024, cfg["levels"], 1e-6)
    assert int(max_rank) == bf_o.max_rank() and int(nbytes) == 16 * bf_o.nnz()
    assert int(cols) == sum(p["forward_columns"] + p["transpose_columns"] for p in log_o["phases"])
    assert float(err) < 1e-5
    lj = json.load(open(tmp_path / "run" / "log.json"))
    assert [p["name"] for p in lj["phases"]] == [p["name"] for p in log_o["phases"]]
    assert [p["rounds"] for p in lj["phases"]] == [p["rounds"] for p in log_o["phases"]]
    got = O.HybridButterfly.deserialize(open(tmp_path / "run" / "butterfly.bfh", "rb").read())
    np.testing.assert_array_equal(got.rank_profile(), bf_o.rank_profile())


@pytest.mark.gpu
def test_cli_synth_container_is_the_references_generator(tmp_path):
    from paper_2002_03400_b200 import cli

    assert cli.main(["--out", str(tmp_path), "--seed", "7", "synth", "--levels", "4", "--rank", "3"]) == 0
    data = open(tmp_path / "butterfly.bfh", "rb").read()
    ref = O.synth_butterfly(4, 3, 7, real=True)
    got = O.HybridButterfly.deserialize(data)  # parses as the reference format
    assert len(data) == len(bytes(ref.serialize()))
    np.testing.assert_array_equal(got.rank_profile(), ref.rank_profile())
    # same seeded generator (operators.hpp:131-178); Householder QR round-off only
    assert np.abs(got.to_dense() - ref.to_dense()).max() <= 1e-13 * np.abs(ref.to_dense()).max()
    m = json.load(open(tmp_path / "manifest.json"))
    assert (m["n"], m["levels"], m["rank"], m["seed"], m["scalar"]) == (128, 4, 3, 7, "real64")


@pytest.mark.gpu
def test_cli_verify_passes_the_theorem_bounds(tmp_path, capsys):
    from paper_2002_03400_b200 import cli

    cfgp = tmp_path / "cfg.json"
    cfgp.write_text(json.dumps({"operator": "nufft1d", "n": 1024}))
    rc = cli.main(["--eps", "1e-6", "--r0", "16", "verify", "--config", str(cfgp)])
    out = capsys.readouterr().out
    assert rc == 0, out
    lines = out.splitlines()
    L, lm = 5, 2
    assert sum(l.startswith("column-basis bound") for l in lines) == L - lm + 1
    assert sum(l.startswith("row-basis bound") for l in lines) == lm + 1
    assert any(l.startswith("combined bound") for l in lines) and "FAIL" not in out
    assert lines[-1].startswith("relative apply error:")

