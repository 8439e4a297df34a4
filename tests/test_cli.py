"""CLI surface (paper_2206_14148_b200/cli.py) mirroring the reference's
tensorbudget CLI (cli.py:1-248): flags, TB_FLAGS precedence, size literals,
CSV schema, oom rows, exit codes; plus reference-IR graph recognition."""

import csv
import io
import os

import numpy as np
import pytest

from paper_2206_14148_b200 import cli, graph

REF_SRC = "/root/reference/pkg/src"


def run(argv, env=None):
    config, args = cli.parse_config(argv, env=env or {})
    out = io.StringIO()
    rc = (cli.cmd_bench if args.command == "bench" else cli.cmd_verify)(config, args, out)
    return rc, out.getvalue()


def test_flags_env_and_size_literals():
    config, args = cli.parse_config(["bench", "knn", "--tensor-split-size=500MB"],
                                    env={"TB_FLAGS": "--tensor-size-threshold=1GiB "
                                                     "--tensor-split-size=64MiB"})
    assert config.tensor_size_threshold == 2**30
    assert config.tensor_split_size == 500 * 10**6       # explicit flag wins
    with pytest.raises(SystemExit) as e:
        cli.parse_config(["bench", "knn", "--budget", "12XB"], env={})
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:                  # split > threshold
        cli.parse_config(["bench", "knn", "--tensor-size-threshold=1MB",
                          "--tensor-split-size=2MB"], env={})
    assert e.value.code == 2


def test_pairwise_is_a_usage_error():
    with pytest.raises(SystemExit) as e:
        cli.parse_config(["bench", "pairwise"], env={})
    assert e.value.code == 2


def test_bench_over_budget_is_an_oom_row_not_a_crash(tmp_path):
    """The planner rejects the budget before any device work (CPU only)."""
    trace = tmp_path / "trace.csv"
    rc, text = run(["bench", "knn", "-n", "20000", "-m", "64", "-d", "16",
                    "--budget", "100KB", "--repeats", "2", "--trace-csv", str(trace)])
    assert rc == 0
    rows = list(csv.reader(io.StringIO(text)))
    assert tuple(rows[0]) == cli._CSV_HEADER
    assert [r[12] for r in rows[1:]] == ["oom", "oom"]
    assert rows[1][:7] == ["knn", "20000", "64", "16", "10", "l2", "f64"]
    assert rows[1][10] == "100000"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
def test_reference_ir_graphs_are_recognised():
    import sys
    sys.path.insert(0, REF_SRC)
    import tensorbudget as ref
    g = graph.from_reference(ref.build_knn(500, 20, 6, 4, "cosine", ref.DType.F32))
    assert (g.kind, g.attrs["metric"], g.attrs["n"], g.attrs["k"]) == ("knn", "cosine", 500, 4)
    assert g.parameters[0].dtype is graph.DType.F32
    gp = ref.run_pipeline(ref.build_knn(5000, 20, 6, 4), ref.PassConfig(tensor_size_threshold=10**5))
    assert graph.from_reference(gp).attrs["dtype"] is graph.DType.F64
    for g in (ref.build_kernel_mvm(64, ref.KernelSpec(1.7, 0.45)),
              ref.run_pipeline(ref.build_kernel_mvm(64, ref.KernelSpec(1.7, 0.45)),
                               ref.PassConfig(tensor_size_threshold=4000))):
        s = graph.from_reference(g).attrs["spec"]
        assert s.variance == 1.7 and abs(s.lengthscale - 0.45) < 1e-15
    with pytest.raises(graph.EvaluationError):
        graph.from_reference(ref.build_pairwise_distance(10, 10, 2))


@pytest.mark.gpu
@pytest.mark.parametrize("argv", [
    ["bench", "knn", "-n", "20000", "-m", "300", "-d", "32", "--dtype", "f32", "--repeats", "2"],
    ["bench", "knn", "-n", "5000", "-m", "40", "-d", "8", "--metric", "l1"],
    ["bench", "mvm", "-n", "3000", "--variance", "1.3", "--lengthscale", "0.4"]])
def test_bench_rows_on_the_gpu(argv):
    rc, text = run(argv)
    rows = list(csv.reader(io.StringIO(text)))
    assert rc == 0 and all(r[12] == "ok" and int(r[13]) > 0 for r in rows[1:])
    if argv[1] == "knn":
        assert float(rows[1][15]) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("argv", [
    ["verify", "knn", "-n", "8000", "-m", "64", "-d", "16", "--seeds", "2"],
    ["verify", "knn", "-n", "8000", "-m", "64", "-d", "16", "--metric", "cosine",
     "--dtype", "f32", "--seeds", "2"],
    ["verify", "knn", "-n", "6000", "-m", "32", "-d", "8", "--metric", "l1", "--seeds", "2"],
    ["verify", "mvm", "-n", "2000", "--seeds", "2"]])
def test_verify_passes_on_the_gpu(argv):
    rc, text = run(argv)
    assert rc == 0 and text.strip().splitlines()[-1].startswith("PASS"), text
