"""Generate tests/golden/formats/ FROM THE REFERENCE ITSELF.

The unmodified reference writers (vsp::write_tensor, save_checkpoint, write_indices via
oracle/_ref/libvspref.so) produce the binary/text files, and the reference readers record
what they return — or the exception type and text they throw — for a corpus of valid and
malformed inputs (the reference's own TensorIo / Checkpoint / IndicesText cases plus
stream-parsing edge cases). tests/test_formats.py checks csrc/formats.cpp against these on
machines without /root/reference. Re-run here with:

    make -C oracle && python tests/golden/make_format_golden.py
"""
from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "formats")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

# Index-text corpus: the reference's IndicesText cases (test_sparsity.cpp:253-312) and
# edge cases of its `std::istringstream >> long long` parsing.
INDEX_TEXTS = [
    "V: 1 3 17\nS: 0 5\n", "V:\nS: 0\n", "V: 2 4\r\nS: 0 1\r\n", "", "X: 1\nS: 0\n", "V: 1\n",
    "V: -1\nS: 0\n", "V: 3 3\nS: 0\n", "V: 1 x\nS: 0\n", "V:5\nS:0", "V: +5\nS: 0\n", "V: -0 1\nS: 0\n",
    "V: 1 -\nS: 0\n", "V: 1 - 2\nS: 0\n", "V: 99999999999999999999\nS: 0\n",
    "V: 99999999999999999999 1\nS: 0\n", "V: 1\t2  3 \nS:  0\n", "V: 1\n\nS: 0\n", "V: 1\nS: 0 4 2\n",
    "V: 1\nS: 0\nextra line\n", "V: 7abc\nS: 0\n", "V: 1\r\r\nS: 0\n", "v: 1\nS: 0\n", "V: 9223372036854775807\nS:\n",
    "V: 0 1 2 3 4 5 6 7 8 9 10 11 12 13 14 15\nS: 0 3 100000\n", "V: 1.5\nS: 0\n", "V: 0x10\nS: 0\n",
]


def main():
    ref = oracle.ref_formats()
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    rng = np.random.default_rng(20260305)
    manifest = {"source": "reference vsp:: writers/readers via oracle/_ref (ref_shim.cpp)", "files": {},
                "index_texts": [], "tensor_errors": [], "checkpoint_errors": []}

    # --- files written by the reference
    m = rng.standard_normal((5, 3))
    v = np.array([1.5, -2.25, 0.0, 1e-300, 1e300])
    assert ref.write_matrix(os.path.join(OUT, "matrix_5x3.vstn"), m)[0] == "ok"
    assert ref.write_vector(os.path.join(OUT, "vector_5.vstn"), v)[0] == "ok"
    assert ref.write_vector(os.path.join(OUT, "vector_1.vstn"), [1.0])[0] == "ok"
    assert ref.write_matrix(os.path.join(OUT, "matrix_0x4.vstn"), np.zeros((0, 4)))[0] == "ok"
    manifest["files"]["matrix_5x3.vstn"] = {"kind": "matrix", "data": m.tolist()}
    manifest["files"]["vector_5.vstn"] = {"kind": "vector", "data": v.tolist()}
    manifest["files"]["vector_1.vstn"] = {"kind": "vector", "data": [1.0]}
    manifest["files"]["matrix_0x4.vstn"] = {"kind": "matrix", "shape": [0, 4], "data": []}

    ck = {"w_u": rng.uniform(-0.35, 0.35, (8, 5)), "b_u": rng.standard_normal(5), "w_v": rng.standard_normal(5),
          "b_v": 0.25, "w_s": rng.standard_normal(5), "b_s": -1.5}
    assert ref.save_checkpoint(os.path.join(OUT, "indexer_d4_dh5.vsck"), **ck)[0] == "ok"
    manifest["files"]["indexer_d4_dh5.vsck"] = {"kind": "checkpoint",
                                               **{k: (x.tolist() if hasattr(x, "tolist") else x) for k, x in ck.items()}}
    for name, iv, is_ in [("indices_a.txt", [1, 3, 17], [0, 5]), ("indices_empty_v.txt", [], [0]),
                          ("indices_big.txt", sorted(rng.choice(1 << 20, 300, replace=False).tolist()),
                           [0] + sorted(rng.choice(np.arange(1, 1 << 17), 40, replace=False).tolist()))]:
        assert ref.write_indices(os.path.join(OUT, name), iv, is_)[0] == "ok"
        manifest["files"][name] = {"kind": "indices", "i_v": [int(x) for x in iv], "i_s": [int(x) for x in is_]}

    tmp = tempfile.mkdtemp()
    try:
        # --- index text parsing
        for text in INDEX_TEXTS:
            p = os.path.join(tmp, "idx.txt")
            with open(p, "wb") as f:
                f.write(text.encode())
            kind, val = ref.read_indices(p)
            manifest["index_texts"].append({"text": text, "kind": kind, "value": val})

        # --- tensor reader errors (the path is part of the message: stored as {path})
        def tcase(name, data: bytes, rank):
            p = os.path.join(tmp, name)
            with open(p, "wb") as f:
                f.write(data)
            kind, val = ref.read(p, rank)
            if kind != "ok":
                val = val.replace(p, "{path}")
            else:
                val = val.tolist()
            manifest["tensor_errors"].append({"name": name, "bytes": data.hex(), "rank": rank, "kind": kind,
                                              "value": val})

        good_v = open(os.path.join(OUT, "vector_5.vstn"), "rb").read()
        good_m = open(os.path.join(OUT, "matrix_5x3.vstn"), "rb").read()
        tcase("badmagic.vstn", b"JUNKxxxxxxxxxxxx", 2)
        tcase("trunc.vstn", b"VS", 2)
        tcase("trunc_dims.vstn", good_m[:14], 2)
        tcase("short_payload.vstn", good_v[:28], 1)
        tcase("version9.vstn", good_v[:4] + bytes([9, 0, 0, 0]) + good_v[8:], 1)
        tcase("rank1_as_matrix.vstn", good_v, 2)
        tcase("rank2_as_vector.vstn", good_m, 1)
        tcase("rank3_as_matrix.vstn", b"VSTN" + (1).to_bytes(4, "little") + (3).to_bytes(4, "little") +
              b"".join(x.to_bytes(8, "little") for x in (1, 1, 1)) + np.float64(2.0).tobytes(), 2)
        tcase("empty.vstn", b"", 1)
        missing = os.path.join(tmp, "missing.vstn")
        kind, val = ref.read(missing, 2)
        manifest["tensor_errors"].append({"name": "missing.vstn", "bytes": None, "rank": 2, "kind": kind,
                                          "value": val.replace(missing, "{path}")})

        # --- checkpoint reader errors
        good_c = open(os.path.join(OUT, "indexer_d4_dh5.vsck"), "rb").read()

        def ccase(name, data):
            p = os.path.join(tmp, name)
            if data is not None:
                with open(p, "wb") as f:
                    f.write(data)
            kind, val = ref.load_checkpoint(p)
            if kind == "ok":
                val = None
            else:
                val = val.replace(p, "{path}")
            manifest["checkpoint_errors"].append({"name": name, "bytes": None if data is None else data.hex(),
                                                  "kind": kind, "value": val})

        ccase("bad_magic.vsck", b"NOPE then some bytes")
        ccase("cut.vsck", good_c[:len(good_c) // 2])
        ccase("header_only.vsck", good_c[:14])
        ccase("version2.vsck", good_c[:4] + bytes([2, 0, 0, 0]) + good_c[8:])
        ccase("missing.vsck", None)
    finally:
        shutil.rmtree(tmp)

    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
