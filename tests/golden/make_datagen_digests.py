"""Record the reference's own `gen` output for the harness restatement.

Runs the UNMODIFIED reference generator (pdqsort.datagen.generate, R/pkg/src/pdqsort/datagen.py:140-157)
in the build container, where /root/reference exists, for every distribution kind over a grid of
sizes and seeds, and writes the input digests (datagen.array_digest, datagen.py:160-163) plus a few
full small arrays and a `gen` file to tests/golden/datagen_digests.json.  The GPU box never runs
this script; tests/test_harness_cpu.py compares paper_2106_05123_b200.harness against the file.

Usage:  python tests/golden/make_datagen_digests.py
"""

from __future__ import annotations

import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from pdqsort import datagen  # noqa: E402  (the reference, imported read-only)

SIZES = (0, 1, 2, 3, 7, 8, 64, 100, 1000, 4096, 65536, 1 << 20)
SEEDS = (0, 1, 0xDE5C)


def main():
    digests = []
    for kind in datagen.DISTRIBUTION_KINDS:
        for n in SIZES:
            for seed in SEEDS:
                if n == 1 << 20 and seed != 0xDE5C:
                    continue
                vals = datagen.generate(datagen.DistributionSpec(kind, n, "int64", seed=seed))
                digests.append({"kind": kind, "n": n, "seed": seed, "digest": datagen.array_digest(vals)})
    arrays = []
    for kind in datagen.DISTRIBUTION_KINDS:
        arrays.append({"kind": kind, "n": 37, "seed": 5,
                       "values": datagen.generate(datagen.DistributionSpec(kind, 37, "int64", seed=5))})
    buf = io.StringIO()
    spec = datagen.DistributionSpec("mod8", 10, "int64", seed=3)
    datagen.write_array(buf, spec, datagen.generate(spec))
    out = {"source": "R/pkg/src/pdqsort/datagen.py (generate, array_digest, write_array)",
           "digests": digests, "arrays": arrays, "gen_file_mod8_10_seed3": buf.getvalue()}
    with open(os.path.join(HERE, "datagen_digests.json"), "w") as f:
        json.dump(out, f, indent=0)
        f.write("\n")
    print(f"{len(digests)} digests")


if __name__ == "__main__":
    main()
