"""Harness integration on the B200: the `gpu` algorithm through the
reference's benchmark table and `gen` files, outputs checked against numpy's sort of the same
generated input, input hashes against the reference's own generator digests."""

import csv
import io
import json
import os

import numpy as np
import pytest

from paper_2106_05123_b200 import harness as h

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = {(e["kind"], e["n"], e["seed"]): e["digest"]
        for e in json.load(open(os.path.join(HERE, "golden", "datagen_digests.json")))["digests"]}


def test_bench_matrix_csv(tmp_path):
    out = tmp_path / "out.csv"
    rc = h.main(["bench", "--out", str(out), "--min-time", "0s", "--min-iters", "2", "--algos", "gpu",
                 "--sizes", "0,1,7,64,1000,65536", "--types", "int64,int32,float32,float64", "--seed", "1"])
    assert rc == 0
    text = out.read_text()
    assert text.splitlines()[0] == ",".join(h.CSV_COLUMNS)
    rows = list(csv.DictReader(io.StringIO(text)))
    assert len(rows) == 12 * 6 * 4
    for r in rows:
        assert r["algo"] == "gpu" and int(r["iterations"]) >= 2
        key = (r["kind"], int(r["n"]), 1)
        if r["element_type"] in ("int64", "int32") and key in GOLD:
            assert r["input_hash"] == GOLD[key], key
        if r["kind"] in ("asc", "desc", "ones") and int(r["n"]) > 1:
            assert int(r["partition_right_calls"]) == 0, r  # K4: one pass, no partitions


def test_bench_outputs_sorted_per_cell():
    # run_benchmark(verify=True) compares every counter-pass output with numpy's sort
    specs = [h.DistributionSpec(k, 1 << 20, "int64", h.DEFAULT_SEED) for k in h.DISTRIBUTION_KINDS]
    recs = h.run_benchmark(["gpu"], specs, h.BenchPolicy(0.0, 1))
    for r in recs:
        assert r.input_hash == GOLD[(r.kind, r.n, h.DEFAULT_SEED)]
        assert r.metrics.max_depth >= 0
    by = {r.kind: r for r in recs}
    assert by["mod8"].metrics.partition_left_calls > 0  # equal-key split (K3) on 8 distinct keys
    assert by["uniform"].metrics.partition_right_calls > 0


def test_sort_gen_file(tmp_path):
    src, dst = tmp_path / "in.txt", tmp_path / "out.txt"
    assert h.main(["gen", "--kind", "organ", "--n", "50000", "--type", "float32", "--seed", "4",
                   "--out", str(src)]) == 0
    assert h.main(["sort", str(src), "--out", str(dst)]) == 0
    with open(src) as f:
        _, before = h.read_array(f)
    with open(dst) as f:
        spec, after = h.read_array(f)
    assert spec.kind == "organ" and spec.element_type == "float32"
    assert list(after) == sorted(before)


def test_instrumented_leg_sorts_in_place():
    spec = h.DistributionSpec("uniform", 300000, "int64", 2)
    vals = h.generate(spec)
    m = h.instrumented_gpu(vals)
    assert vals == np.sort(h.generate_values(spec)).tolist()
    assert m.partition_right_calls > 0 and m.comparisons == 0
