"""Relation-file fixtures from the REFERENCE's own bench.write_relation /
bench.read_relation (/root/reference/pkg/src/mpsm/bench.py:73-102).

    python tests/golden/make_relfile_golden.py

Writes tests/golden/rel_small.mpsmrel (a 256-tuple relation written by the
reference) and tests/golden/relfile.json: the relation's keys/payloads and,
for malformed variants of the file, the FormatError message (path replaced
by {path}) and byte_offset the reference raises.  Runs in the build
container only (the reference is absent on the GPU box).
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

from mpsm import bench as rbench  # noqa: E402  (the reference)
from mpsm.core import FormatError, KeyDomain  # noqa: E402
from mpsm.datagen import GenSpec, generate  # noqa: E402

# malformed variants: (name, how to derive the bytes from the good file)
VARIANTS = {
    "bad_magic": lambda b: b"MPSMREL2" + b[8:],
    "short_magic": lambda b: b[:5],
    "truncated_header": lambda b: b[:12],
    "extra_byte": lambda b: b + b"\x00",
    "missing_record": lambda b: b[:-16],
    "missing_byte": lambda b: b[:-1],
    "count_too_large": lambda b: b[:8] + (10**6).to_bytes(8, "little") + b[16:],
    "empty_file": lambda b: b"",
}


def main():
    rel = generate(GenSpec(256, KeyDomain(0, 1 << 40), "uniform", seed=7))
    good = os.path.join(HERE, "rel_small.mpsmrel")
    rbench.write_relation(rel, good)
    blob = open(good, "rb").read()
    out = {"n": int(rel.cardinality), "keys": [int(x) for x in rel.keys], "payloads": [int(x) for x in rel.payloads],
           "file_bytes": len(blob), "errors": {}}
    with tempfile.TemporaryDirectory() as td:
        for name, fn in VARIANTS.items():
            p = os.path.join(td, name)
            with open(p, "wb") as fh:
                fh.write(fn(blob))
            try:
                rbench.read_relation(p)
                out["errors"][name] = None
            except FormatError as exc:
                out["errors"][name] = {"message": str(exc).replace(p, "{path}"), "byte_offset": exc.byte_offset}
        # zero-tuple file written by the reference
        from mpsm.core import Relation
        import numpy as np
        p = os.path.join(td, "zero")
        rbench.write_relation(Relation(np.zeros(0, np.uint64), np.zeros(0, np.uint64)), p)
        out["zero_file_hex"] = open(p, "rb").read().hex()
    with open(os.path.join(HERE, "relfile.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print({k: v for k, v in out["errors"].items()})


if __name__ == "__main__":
    main()
