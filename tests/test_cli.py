"""The command-line tool end to end (tests/test_cli.cpp restated): exit codes,
output formats, cache round trip, index determinism, groundtruth and the
sweep harness. Commands that run queries need the GPU; argument and
data-error paths that fail before any device work run on CPU."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIVE = "# five-node example\n0 1\n0 2\n1 0\n1 2\n1 3\n1 4\n2 1\n2 3\n3 0\n3 1\n3 2\n4 1\n4 2\n"


def run(*args):
    p = subprocess.run([sys.executable, "-m", "paper_2101_03652_b200", *args], cwd=ROOT,
                       capture_output=True, text=True)
    return p.returncode, p.stdout, p.stderr


@pytest.fixture
def graph(tmp_path):
    p = tmp_path / "graph.txt"
    p.write_text(FIVE)
    return str(p)


def slurp(p):
    with open(p, "rb") as f:
        return f.read()


def test_usage_errors_exit_1(graph):
    assert run()[0] == 1                                             # missing subcommand
    assert run("query", "--graph", graph, "--algo", "nosuch", "--source", "0")[0] == 1
    assert run("query", "--graph", graph, "--algo", "speedppr", "--source", "0")[0] == 1
    assert run("query", "--graph", graph, "--algo", "powerpush", "--source", "0",
               "--random-sources", "3")[0] == 1
    assert run("bench", "--graph", graph, "--algo", "nosuch", "--source", "0")[0] == 1
    assert run("--help")[0] == 0


def test_data_errors_exit_2(tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("0 1\nnot an edge\n")
    rc, _, err = run("query", "--graph", str(bad), "--algo", "powerpush", "--source", "0")
    assert rc == 2 and "bad.txt:2: expected non-negative integer source id" in err
    assert run("query", "--graph", "/nonexistent.txt", "--algo", "powerpush",
               "--source", "0")[0] == 2


def test_edge_list_parser_rules(tmp_path):
    from paper_2101_03652_b200.formats import parse_edge_list
    from paper_2101_03652_b200 import DataError
    p = tmp_path / "e.txt"
    p.write_text("  # c\n\n0\t1\r\n 7 3 \n")
    e = parse_edge_list(str(p))
    assert e.tolist() == [[0, 1], [7, 3]]
    assert parse_edge_list(str(p), undirected=True).tolist() == [[0, 1], [1, 0], [7, 3], [3, 7]]
    for text, msg in (("1 2 3\n", ":1: trailing content after edge pair"),
                      ("1 x\n", ":1: expected non-negative integer target id"),
                      ("-1 2\n", ":1: expected non-negative integer source id"),
                      ("# only\n", "graph is empty after cleaning")):
        p.write_text(text)
        with pytest.raises(DataError, match=msg):
            parse_edge_list(str(p))


@pytest.mark.gpu
def test_cli_end_to_end(graph, tmp_path):
    t = lambda name: str(tmp_path / name)  # noqa: E731
    rc, out, _ = run("query", "--graph", graph, "--algo", "powerpush", "--source", "0",
                     "--out", t("result.csv"))
    assert rc == 0 and out.startswith("algorithm,param,edge_pushes,wall_time_ns,achieved_r_sum\n")
    lines = slurp(t("result.csv")).decode().splitlines()
    assert lines[0] == "node,ppr" and len(lines) == 6
    for algo in ("powitr", "simfwdpush", "fwdpush-fifo"):
        assert run("query", "--graph", graph, "--algo", algo, "--random-sources", "2",
                   "--seed", "1", "--out", t(algo + ".csv"))[0] == 0
    # clean -> cache -> the same bytes
    rc, out, _ = run("clean", "--graph", graph, "--out", t("g.pprg"))
    assert rc == 0 and out.strip() == "n=5 m=13 dead_ends=0"
    assert run("query", "--graph", t("g.pprg"), "--algo", "powerpush", "--source", "0",
               "--out", t("from_cache.csv"))[0] == 0
    assert slurp(t("from_cache.csv")) == slurp(t("result.csv"))
    # speedppr: same argv, same bytes
    for name in ("s2.csv", "s3.csv"):
        assert run("query", "--graph", graph, "--algo", "speedppr", "--epsilon", "0.5",
                   "--seed", "7", "--source", "0", "--out", t(name))[0] == 0
    assert slurp(t("s2.csv")) == slurp(t("s3.csv"))
    # build-index deterministic; alpha mismatch is a data error
    for name in ("a.pprw", "b.pprw"):
        rc, out, _ = run("build-index", "--graph", graph, "--alpha", "0.2", "--seed", "42",
                         "--out", t(name))
        assert rc == 0 and out.strip() == "endpoints=13"
    assert slurp(t("a.pprw")) == slurp(t("b.pprw")) and len(slurp(t("a.pprw"))) > 0
    assert run("query", "--graph", graph, "--algo", "speedppr", "--epsilon", "0.5", "--alpha",
               "0.15", "--index", t("a.pprw"), "--source", "0")[0] == 2
    assert run("query", "--graph", graph, "--algo", "speedppr", "--epsilon", "0.5", "--seed", "3",
               "--index", t("a.pprw"), "--source", "0", "--out", t("wi.csv"))[0] == 0
    # groundtruth
    assert run("groundtruth", "--graph", graph, "--source", "0", "--out", t("truth.csv"))[0] == 0
    assert slurp(t("truth.csv")).startswith(b"node,ppr\n")
    from paper_2101_03652_b200.harness import read_ppr_csv
    from oracle.pyoracle import FIVE_NODE_PI0
    import numpy as np
    assert np.abs(read_ppr_csv(t("truth.csv")) - FIVE_NODE_PI0).sum() <= 1e-12
    # bench: sweep summary + checkpoint series
    rc, out, _ = run("bench", "--graph", graph, "--algo", "powerpush", "--algo", "speedppr",
                     "--lambda", "1e-6", "--epsilon", "0.5", "--random-sources", "2", "--seed",
                     "1", "--out", t("bench"), "--name", "example")
    assert rc == 0 and out.strip() == "cells=4"
    summary = slurp(t("bench") + "/example_sweep.csv").decode().splitlines()
    assert summary[0] == "source,algo,param,wall_time_ns,edge_pushes,walks,l1_error,max_rel_error"
    assert len(summary) == 5
