"""CPU: the interchange formats behind the C ABI (csrc/formats.cpp) against the reference.

1. Files the reference wrote (tests/golden/formats/, make_format_golden.py): our writers
   produce them byte for byte and our readers read them exactly.
2. The reference readers' verdicts (value, or exception type + text) on a corpus of valid
   and malformed files (manifest.json) — the TensorIo / Checkpoint / IndicesText suites
   (test_config.cpp:140-229, test_indexer.cpp:487-547, test_sparsity.cpp:253-312).
3. Live differential against oracle/_ref on random inputs when it is built here.
No GPU: these are host files; the C-ABI library loads without a device.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2603_04460_b200 import IndexerParams, VspError, VspRuntimeError
from paper_2603_04460_b200 import formats as fm

GOLD = os.path.join(os.path.dirname(__file__), "golden", "formats")
MAN = json.load(open(os.path.join(GOLD, "manifest.json")))


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


def _expect(kind, msg, fn):
    exc = VspRuntimeError if kind == "runtime_error" else VspError
    with pytest.raises(exc) as ei:
        fn()
    assert str(ei.value) == msg


# --------------------------------------------------------------------------- golden files

@pytest.mark.parametrize("name", sorted(MAN["files"]))
def test_reader_reads_reference_files(name):
    spec = MAN["files"][name]
    path = os.path.join(GOLD, name)
    if spec["kind"] == "matrix":
        got = fm.read_tensor(path)
        want = np.array(spec["data"], dtype=np.float64).reshape(spec.get("shape", np.shape(spec["data"])))
        assert got.shape == want.shape and np.array_equal(got, want)
    elif spec["kind"] == "vector":
        got = fm.read_vector(path)
        assert got.tolist() == spec["data"]  # exact, including 1e-300 and 1e300
    elif spec["kind"] == "checkpoint":
        ck = fm.load_checkpoint(path)
        assert ck["d_h"] == len(spec["b_u"])
        for key in ("w_u", "b_u", "w_v", "w_s"):
            assert np.array_equal(ck[key], np.array(spec[key]))
        assert ck["b_v"] == spec["b_v"] and ck["b_s"] == spec["b_s"]
    else:
        assert fm.read_indices(path) == (spec["i_v"], spec["i_s"])


@pytest.mark.parametrize("name", sorted(MAN["files"]))
def test_writer_matches_reference_bytes(name, tmp_path):
    spec = MAN["files"][name]
    out = tmp_path / name
    if spec["kind"] in ("matrix", "vector"):
        data = np.array(spec["data"], dtype=np.float64)
        if spec["kind"] == "matrix":
            data = data.reshape(spec.get("shape", data.shape))
        fm.write_tensor(out, data)
    elif spec["kind"] == "checkpoint":
        fm.save_checkpoint({k: spec[k] for k in ("w_u", "b_u", "w_v", "b_v", "w_s", "b_s")}, out)
    else:
        fm.write_indices(out, spec["i_v"], spec["i_s"])
    assert _bytes(out) == _bytes(os.path.join(GOLD, name))


# --------------------------------------------------------------------------- reference KATs

def test_tensor_header_layout_is_stable(tmp_path):
    # test_config.cpp:172-191: magic, version=1, ndim=1, dim=1, one f64 -> 28 bytes
    p = tmp_path / "h.vstn"
    fm.write_tensor(p, np.array([1.0]))
    b = _bytes(p)
    assert len(b) == 28 and b[:4] == b"VSTN" and b[4] == 1 and b[8] == 1 and b[12] == 1


def test_tensor_round_trips_are_exact(tmp_path):
    # test_config.cpp:140-170
    m = np.random.default_rng(121).standard_normal((5, 3))
    fm.write_tensor(tmp_path / "m.vstn", m)
    assert np.array_equal(fm.read_tensor(tmp_path / "m.vstn"), m)
    v = np.array([1.5, -2.25, 0.0, 1e-300, 1e300])
    fm.write_tensor(tmp_path / "v.vstn", v)
    assert fm.read_vector(tmp_path / "v.vstn").tolist() == v.tolist()
    with pytest.raises(VspRuntimeError):
        fm.read_tensor(tmp_path / "v.vstn")
    with pytest.raises(VspRuntimeError):
        fm.read_vector(tmp_path / "m.vstn")
    # any-rank extension and torch input (bf16 widens exactly)
    t = torch.randn(2, 3, 4).bfloat16()
    fm.write_tensor(tmp_path / "t.vstn", t)
    assert fm.tensor_shape(tmp_path / "t.vstn") == (2, 3, 4)
    assert np.array_equal(fm.read_tensor_any(tmp_path / "t.vstn"), t.double().numpy())


@pytest.mark.parametrize("case", MAN["tensor_errors"], ids=lambda c: c["name"])
def test_tensor_reader_errors_match_reference(case, tmp_path):
    p = tmp_path / case["name"]
    if case["bytes"] is not None:
        p.write_bytes(bytes.fromhex(case["bytes"]))
    fn = (lambda: fm.read_tensor(p)) if case["rank"] == 2 else (lambda: fm.read_vector(p))
    if case["kind"] == "ok":
        assert fn().tolist() == case["value"]
    else:
        _expect(case["kind"], case["value"].replace("{path}", str(p)), fn)


@pytest.mark.parametrize("case", MAN["checkpoint_errors"], ids=lambda c: c["name"])
def test_checkpoint_errors_match_reference(case, tmp_path):
    # test_indexer.cpp:503-547 (foreign, truncated, missing, "unsupported VSCK version 2")
    p = tmp_path / case["name"]
    if case["bytes"] is not None:
        p.write_bytes(bytes.fromhex(case["bytes"]))
    _expect(case["kind"], case["value"].replace("{path}", str(p)), lambda: fm.load_checkpoint(p))


def test_checkpoint_round_trip_is_exact(tmp_path):
    # test_indexer.cpp:487-501
    rng = np.random.default_rng(83)
    ck = {"w_u": rng.uniform(-0.35, 0.35, (8, 5)), "b_u": np.zeros(5), "w_v": rng.standard_normal(5),
          "b_v": 0.25, "w_s": rng.standard_normal(5), "b_s": -1.5}
    fm.save_checkpoint(ck, tmp_path / "c.vsck")
    back = fm.load_checkpoint(tmp_path / "c.vsck")
    for k in ("w_u", "b_u", "w_v", "w_s"):
        assert np.array_equal(back[k], ck[k])
    assert back["b_v"] == 0.25 and back["b_s"] == -1.5 and back["d_h"] == 5
    with pytest.raises(VspError, match="in_dim must be 2d"):
        fm.save_checkpoint({**ck, "w_u": np.zeros((7, 5))}, tmp_path / "odd.vsck")
    with pytest.raises(VspError, match="inconsistent shapes"):
        fm.save_checkpoint({**ck, "b_u": np.zeros(4)}, tmp_path / "bad.vsck")


def test_checkpoints_drive_the_device_params(tmp_path):
    """IndexerParams -> one VSCK per KV head -> IndexerParams: W_U (bf16) survives exactly;
    the heads go through f64 and back to fp32 exactly."""
    g = torch.Generator().manual_seed(5)
    hkv, d, dh = 2, 4, 6
    p = IndexerParams(torch.randn(hkv, 2 * d, dh, generator=g).bfloat16(), torch.randn(hkv, dh, generator=g),
                      torch.randn(hkv, dh, generator=g), torch.randn(hkv, generator=g),
                      torch.randn(hkv, dh, generator=g), torch.randn(hkv, generator=g))
    paths = [tmp_path / f"h{t}.vsck" for t in range(hkv)]
    fm.save_checkpoints(p, paths)
    q = fm.load_checkpoints(paths, device="cpu")
    for a, b in zip((p.w_u, p.b_u, p.w_v, p.b_v, p.w_s, p.b_s), (q.w_u, q.b_u, q.w_v, q.b_v, q.w_s, q.b_s)):
        assert a.dtype == b.dtype and torch.equal(a, b)


@pytest.mark.parametrize("case", MAN["index_texts"], ids=lambda c: repr(c["text"])[:40])
def test_index_text_parsing_matches_reference(case, tmp_path):
    p = tmp_path / "idx.txt"
    p.write_bytes(case["text"].encode())
    if case["kind"] == "ok":
        assert list(fm.read_indices(p)) == case["value"]
    else:
        _expect(case["kind"], case["value"], lambda: fm.read_indices(p))


def test_index_text_round_trip_and_missing_file(tmp_path):
    # test_sparsity.cpp:253-277, 311
    fm.write_indices(tmp_path / "a.txt", [1, 3, 17], [0, 5])
    assert _bytes(tmp_path / "a.txt") == b"V: 1 3 17\nS: 0 5\n"
    assert fm.read_indices(tmp_path / "a.txt") == ([1, 3, 17], [0, 5])
    fm.write_indices(tmp_path / "b.txt", [], [0])
    assert fm.read_indices(tmp_path / "b.txt") == ([], [0])
    with pytest.raises(VspRuntimeError, match="cannot open indices file: /nonexistent/vsp_indices.txt"):
        fm.read_indices("/nonexistent/vsp_indices.txt")


def test_patterns_from_files_builds_device_layout(tmp_path):
    fm.write_indices(tmp_path / "g0.txt", [0, 4, 9], [0, 1])
    fm.write_indices(tmp_path / "g1.txt", [], [0, 2, 3])
    pat = fm.patterns_from_files([tmp_path / "g0.txt", tmp_path / "g1.txt"], n=16, device="cpu")
    assert pat.k_v.tolist() == [3, 0] and pat.k_s.tolist() == [2, 3]
    assert pat.lists(0) == ([0, 4, 9], [0, 1]) and pat.lists(1) == ([], [0, 2, 3])


# --------------------------------------------------------------------------- live differential

@pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built (reference headers absent)")
def test_random_files_agree_with_live_reference(tmp_path):
    ref = oracle.ref_formats()
    rng = np.random.default_rng(7)
    for t in range(20):
        shape = tuple(int(x) for x in rng.integers(0, 7, size=2))
        m = rng.standard_normal(shape) * 10.0 ** rng.integers(-300, 300)
        ref.write_matrix(str(tmp_path / "r.vstn"), m)
        fm.write_tensor(tmp_path / "o.vstn", m)
        assert _bytes(tmp_path / "r.vstn") == _bytes(tmp_path / "o.vstn")
        iv = np.unique(rng.integers(0, 1 << 40, size=int(rng.integers(0, 30))))
        is_ = np.unique(rng.integers(0, 1 << 20, size=int(rng.integers(0, 30))))
        ref.write_indices(str(tmp_path / "r.txt"), iv, is_)
        fm.write_indices(tmp_path / "o.txt", iv, is_)
        assert _bytes(tmp_path / "r.txt") == _bytes(tmp_path / "o.txt")
        dh = int(rng.integers(1, 9))
        ck = {"w_u": rng.standard_normal((2 * int(rng.integers(1, 5)), dh)), "b_u": rng.standard_normal(dh),
              "w_v": rng.standard_normal(dh), "b_v": float(rng.standard_normal()), "w_s": rng.standard_normal(dh),
              "b_s": float(rng.standard_normal())}
        ref.save_checkpoint(str(tmp_path / "r.vsck"), **ck)
        fm.save_checkpoint(ck, tmp_path / "o.vsck")
        assert _bytes(tmp_path / "r.vsck") == _bytes(tmp_path / "o.vsck")
    # fuzzed index text: same verdict as the reference's stream parser
    alphabet = list("0123456789 +-\t\rxV:S.") + ["\n"]
    for t in range(300):
        body = "".join(rng.choice(alphabet, size=int(rng.integers(0, 14))))
        text = "V:" + body + "\nS: 0" + ("\n" if t % 2 else "")
        p = tmp_path / "f.txt"
        p.write_bytes(text.encode())
        kind, val = ref.read_indices(str(p))
        if kind == "ok":
            assert list(fm.read_indices(p)) == list(val), repr(text)
        else:
            _expect(kind, val, lambda: fm.read_indices(p))
