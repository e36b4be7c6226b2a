"""Harness integration, CPU side: the datagen restatement against the
reference's own generator output (tests/golden/datagen_digests.json, made by
tests/golden/make_datagen_digests.py from R/pkg/src/pdqsort/datagen.py), the `gen` file format,
the CSV schema (golden header of R/pkg/tests/test_cli.py:10-15) and the CLI's usage errors.
No kernel runs here."""

import array
import csv
import io
import json
import os

import pytest

from paper_2106_05123_b200 import harness as h

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "datagen_digests.json")))

# R/pkg/tests/test_cli.py:10-15
GOLDEN_HEADER = (
    "algo,kind,element_type,n,seed,iterations,total_ns,ns_per_nlog2n,input_hash,"
    "comparisons,element_moves,exchanges,partition_right_calls,partition_left_calls,"
    "bad_partitions,heapsort_fallbacks,partial_insertion_attempts,"
    "partial_insertion_aborts,max_depth"
)


@pytest.mark.parametrize("kind", h.DISTRIBUTION_KINDS)
def test_datagen_matches_reference_digests(kind):
    cases = [e for e in GOLD["digests"] if e["kind"] == kind]
    assert len(cases) >= 30
    for e in cases:
        vals = h.generate(h.DistributionSpec(kind, e["n"], "int64", e["seed"]))
        assert h.array_digest(vals) == e["digest"], (kind, e["n"], e["seed"])


def test_datagen_matches_reference_arrays():
    for a in GOLD["arrays"]:
        assert h.generate(h.DistributionSpec(a["kind"], a["n"], "int64", a["seed"])) == a["values"]


def test_gen_file_is_the_reference_format():
    spec = h.DistributionSpec("mod8", 10, "int64", 3)
    buf = io.StringIO()
    h.write_array(buf, spec, h.generate(spec))
    assert buf.getvalue() == GOLD["gen_file_mod8_10_seed3"]
    spec2, vals = h.read_array(io.StringIO(GOLD["gen_file_mod8_10_seed3"]))
    assert spec2 == spec and vals == h.generate(spec)


@pytest.mark.parametrize("etype", h.ELEMENT_TYPES)
def test_element_types_round_trip(etype, tmp_path):
    spec = h.DistributionSpec("dup8", 300, etype, 11)
    vals = h.generate(spec)
    base = h.generate_values(spec)
    assert [int(v) for v in vals] == base.tolist()
    assert isinstance(vals, array.array) == (etype in ("int32", "float32"))
    p = tmp_path / "a.txt"
    assert h.main(["gen", "--kind", "dup8", "--n", "300", "--type", etype, "--seed", "11", "--out", str(p)]) == 0
    with open(p) as f:
        spec2, vals2 = h.read_array(f)
    assert spec2 == spec and list(vals2) == list(vals)


def test_string_types_are_rejected():
    with pytest.raises(ValueError):
        h.DistributionSpec("uniform", 4, "str")
    assert h.main(["gen", "--kind", "uniform", "--n", "4", "--type", "bigstr"]) == 1


def test_csv_schema_is_the_reference_header():
    assert ",".join(h.CSV_COLUMNS) == GOLDEN_HEADER
    rec = h.BenchmarkRecord("gpu", "asc", "int64", 64, 1, 3, 3000, 0.5, "ab", h.DeviceMetrics(max_depth=2))
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(h.CSV_COLUMNS)
    w.writerow(rec.row())
    rows = list(csv.DictReader(io.StringIO(buf.getvalue())))
    assert rows[0]["ns_per_nlog2n"] == "0.500000" and rows[0]["max_depth"] == "2"


def test_device_metrics_mapping():
    st = {"partition_right_calls": 5, "partition_left_calls": 2, "bad_partitions": 1, "radix_fallbacks": 1,
          "max_depth": 9}
    m = h.DeviceMetrics.from_stats(st)
    assert m.counter_values() == (0, 0, 0, 5, 2, 1, 1, 0, 0, 9)
    assert h.DeviceMetrics.from_stats({}).counter_values() == (0,) * 10


def test_size_and_duration_parsing():
    assert h.parse_sizes("16..128:2") == [16, 32, 64, 128]
    assert h.parse_sizes("1024..1048576:4")[-1] == 1048576
    assert h.parse_sizes("0,5") == [0, 5]
    assert h.parse_duration("250ms") == 0.25 and h.parse_duration("2s") == 2.0
    for bad in ("10..2", "abc", "", "4..8:1"):
        with pytest.raises(h.UsageError):
            h.parse_sizes(bad)


@pytest.mark.parametrize(
    "flags",
    [["--algos", "quantum"], ["--dists", "zipf"], ["--types", "str"], ["--sizes", "10..2"], ["--sizes", "abc"],
     ["--min-time", "fast"], ["--min-iters", "0"]],
)
def test_bench_usage_errors_exit_1(tmp_path, flags):
    assert h.main(["bench", "--out", str(tmp_path / "x.csv"), "--min-time", "0s", "--min-iters", "1"] + flags) == 1


def test_gpu_algorithm_entry_has_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    run, instr = h.GPU_ALGORITHM
    with pytest.raises(RuntimeError):
        run([3, 1, 2])
    with pytest.raises(RuntimeError):
        instr([3, 1, 2])
