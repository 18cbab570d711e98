"""CPU-only checks of the product's host side: the C ABI loads and exports every
declared symbol, the engine protocol / seeding / jumps / buffer / checkpoint
logic reproduce the reference (via its golden vectors and the oracle), and the
fill path refuses to run without a GPU (no CPU fallback)."""
import ctypes
import hashlib
import pathlib
import re

import numpy as np
import pytest
import torch

import paper_2605_05099_b200 as P
from paper_2605_05099_b200 import _lib, engines, serialize, state_io
from oracle import oracle as O

ROOT = pathlib.Path(__file__).resolve().parents[1]


def _h(ws):
    return [int(w, 16) for w in ws]


def test_abi_exports_every_declared_symbol():
    hdr = (ROOT / "include" / "randstream_b200.h").read_text()
    declared = set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", hdr))
    assert {"rs_fill", "rs_fill_streams", "rs_mvn", "rs_init_device", "rs_last_error"} <= declared
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTED) == declared
    assert _lib.lib.rs_abi_version() == 1


def test_catalogue_and_registry():
    cat = state_io.catalogue()
    assert [c["id"] for c in cat][:2] == ["x256++", "x256**"]
    assert len(cat) == 14
    assert engines.normalize("X256**") == "x256**"
    assert engines.normalize(None) == engines.normalize("0") == engines.normalize("") == "x256++simd"
    with pytest.raises(engines.UnknownEngineError):
        engines.normalize("nope")
    for e in engines.ENGINE_IDS:  # every registry engine has a device path
        assert engines.supported(e)
        assert engines.make(e).ID == e


def test_engine_kats_host(golden):
    for k in golden["kats"]:
        eng = engines.make(k["engine"])
        if k["how"] == "set_state":
            eng.set_state(_h(k["words"]))
        else:
            eng.seed_from(_h(k["words"]))
        assert eng.generate(len(k["expect"])) == _h(k["expect"]), k["engine"]


def test_seeding_matches_reference(golden):
    from paper_2605_05099_b200 import seeding
    for s in golden["seeding"]:
        assert seeding.derive_seed_words(9, _h(s["entropy"]), tuple(_h(s["spawn"]))) == _h(s["words"])


def test_create_matches_reference_start_states(golden):
    for rec in golden["fills"]:
        r = state_io.create(rec["engine"], seed=rec["seed"], spawn_key=tuple(rec["spawn"]))
        assert r.get_state() == _h(rec["start_state"]), rec["name"]


def test_jumps_and_advance(golden):
    for j in golden["jumps"]:
        r = state_io.create(j["engine"], seed=[77])
        if "advance" in j:
            r.advance(int(j["advance"]))
        else:
            r.next_u64()
            r.jump(j["k"])
        assert r.get_state() == _h(j["state"]), j
        assert [r.next_u64() for _ in range(5)] == _h(j["next"])
    r = state_io.create("philox", seed=[1])
    before = r.get_state()
    with pytest.raises(ValueError):
        r.jump(32)
    assert "jump unsupported" in state_io.last_error(r)  # read before any successful op clears it
    assert r.get_state() == before
    with pytest.raises(ValueError):
        state_io.create("x256**", seed=[1]).jump(33)


@pytest.mark.parametrize("engine", ["x256**", "x256++", "pcg64", "philox", "sfc64", "ranlux++", "x256++simd",
                                    "x256**simd", "sfc64simd", "x128+", "xoro++", "squares", "cwg128", "chacha20"])
def test_scalar_draws_match_oracle(engine):
    r = state_io.create(engine, seed=[4242])
    o = O.OracleRng(engine, seed=[4242])
    for _ in range(3):
        assert [r.next_u64() for _ in range(100)] == [o.next_u64() for _ in range(100)]
        assert [r.next_u32() for _ in range(77)] == [o.next_u32() for _ in range(77)]
    r.set_full_mantissa(True)
    o.set_full_mantissa(True)
    a = [r.u01() for _ in range(300)]
    b = o.fill("u01", {}, 300).tolist()
    assert a == b
    assert [r.u01f() for _ in range(301)] == [float(x) for x in o.fill("u01f", {}, 301)]
    assert r.get_state() == o.get_state()


def test_set_stream_matches_reference(golden):
    for c in golden["streams"]:
        r = state_io.create(c["engine"], seed=[88])
        r.next_u32()
        r.set_stream(_h(c["words"]))
        assert r.get_state() == _h(c["state"]), c["engine"]
        assert [r.next_u64() for _ in range(20)] == _h(c["next"]), c["engine"]


def test_chacha20_exhaustion():
    """counter.py:209-216: generating past block 2^32 - 1 raises OverflowError."""
    r = state_io.create("chacha20", seed=[5])
    st = r.get_state()
    st[5] = (st[5] & 0xFFFFFFFF) | ((2 ** 32 - 2) << 32)
    r.set_state(st)
    with pytest.raises(OverflowError):
        r.next_u64()  # a refill needs 18 blocks, only 2 remain


def test_raw_bytes_and_set_stream():
    r = state_io.create("pcg64", seed=[3])
    o = O.OracleRng("pcg64", seed=[3])
    raw = r.raw(21)
    words = [o.next_u64() for _ in range(3)]
    assert raw == b"".join(w.to_bytes(8, "little") for w in words)[:21]
    with pytest.raises(ValueError):
        r.raw(-1)
    r.set_stream([5, 6])
    assert r.get_state()[2:] == [5 | 1, 6]
    s = state_io.create("sfc64", seed=[3])
    s.set_stream([1, 2, 3])
    assert s.get_state()[3] == 18
    with pytest.raises(ValueError):
        state_io.create("x256**", seed=[1]).set_stream([1])


def test_checkpoint_roundtrip_mid_buffer():
    r = state_io.create("x256**", seed=[9])
    r.next_u64()
    r.next_u32()
    blob = state_io.to_blob(r)
    c = state_io.from_blob(blob)
    assert c.get_state() == r.get_state()
    assert [c.next_u32() for _ in range(300)] == [r.next_u32() for _ in range(300)]
    with pytest.raises(serialize.BlobError):
        state_io.from_blob(blob[:-1] + bytes([blob[-1] ^ 1]))
    with pytest.raises(serialize.BlobError):
        state_io.from_blob(b"XXXX" + blob[4:])


def test_set_state_validation():
    r = state_io.create("x256**", seed=[1])
    with pytest.raises(ValueError):
        r.set_state([0, 0, 0, 0])
    p = state_io.create("pcg64", seed=[1])
    with pytest.raises(ValueError):
        p.set_state([1, 2, 4, 0])
    q = state_io.create("ranlux++", seed=[1])
    with pytest.raises(ValueError):
        q.set_state([2 ** 64 - 1] * 9)


def test_validation_precedes_consumption():
    r = state_io.create("x256**", seed=[1])
    st = r.get_state()
    for dist, params, n in [("norm", {"var": -1.0}, 5), ("gamma", {}, 5), ("gamma", {"alpha": 0.0}, 3),
                            ("exp", {"beta": 0}, 2), ("u01", {"x": 1}, 2), ("uint64", {"b": -1}, 2)]:
        with pytest.raises(ValueError):
            r.fill(dist, params, n)
        assert r.get_state() == st and r.buffer.words == []
    with pytest.raises(ValueError):
        r.fill("norm", {}, -1)
    with pytest.raises(ValueError):
        r.fill("nosuch", {}, 1)
    assert "unknown" in state_io.last_error(r)
    r.fill("norm", {}, 0)
    assert state_io.last_error(r) == ""


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_fill_without_gpu_fails_loudly():
    r = state_io.create("x256**", seed=[1])
    with pytest.raises(_lib.LibraryError):
        r.fill("norm", {}, 10)


def test_n_zero_is_a_no_op():
    r = state_io.create("x256**", seed=[1])
    r.next_u32()
    snap = r.buffer.capture()
    st = r.get_state()
    out = r.fill("norm", {"var": -5}, 0)  # the reference validates nothing for n == 0
    assert out.numel() == 0 if hasattr(out, "numel") else len(out) == 0
    assert r.get_state() == st and r.buffer.capture() == snap


def test_interleaved_lanes_are_jumped_scalar_lanes():
    """interleave.py:9-13 / pkg/tests/test_engines_kat.py:54-98: lane k = base jumped k*2^253."""
    for simd, base in (("x256++simd", "x256++"), ("x256**simd", "x256**")):
        r = engines.make(simd)
        r.seed_from([11, 22, 33, 44])
        b = engines.make(base)
        b.seed_from([11, 22, 33, 44])
        lanes = []
        st = b.get_state()
        for _ in range(8):
            lane = engines.make(base)
            lane.set_state(st)
            lanes.append(lane.generate(25))
            s = _lib.u64_array(st, 32)
            _lib.check(_lib.lib.rs_engine_jump(engines.NATIVE_ID[base], s, 253))
            st = [int(s[i]) for i in range(4)]
        assert r.generate(200) == [lanes[k][i] for i in range(25) for k in range(8)]
    r = engines.make("sfc64simd")
    r.seed_from([5, 6, 7])
    s = engines.make("sfc64")
    s.seed_from([5, 6, 7])
    a, b_, c, w = s.get_state()
    lanes = []
    for k in range(8):
        lane = engines.make("sfc64")
        lane.set_state([a, b_, c, (w + k * (1 << 61)) & (2 ** 64 - 1)])
        lanes.append(lane.generate(25))
    assert r.generate(200) == [lanes[k][i] for i in range(25) for k in range(8)]


def test_default_engine_is_x256pp_simd():
    r = state_io.create(seed=[2024])
    assert r.engine_id == "x256++simd"
    o = O.OracleRng("x256++simd", seed=[2024])
    assert r.get_state() == o.get_state()


def test_dist_info_host_only():
    """rs_dist_info needs no device: unit, variable-consumption flag and provisioning."""
    from paper_2605_05099_b200 import shard

    i = shard.dist_info(_lib.DIST_IDS["norm"], [0.0, 1.0], [])
    assert (i.unit, i.variable, i.min_seg_len % 72) == (1, 1, 0) and 1.0 < i.words_per_sample < 1.1
    assert list(i.tally_seen) == [1, 0, 0]
    i = shard.dist_info(_lib.DIST_IDS["u01f"], [], [])
    assert (i.unit, i.variable) == (2, 0)
    i = shard.dist_info(_lib.DIST_IDS["gamma"], [2.5, 1.0], [])
    assert i.variable == 1 and i.min_seg_len >= 288 and list(i.tally_seen) == [1, 0, 1]
    with pytest.raises(ValueError):
        shard.dist_info(_lib.DIST_IDS["gamma"], [-1.0, 1.0], [])


def test_range_abi_validates_before_touching_a_device():
    """rs_range_count checks its inputs before any CUDA call (reference rule: validation
    first, src/continuous.py:413-431), so these run without a GPU."""
    import ctypes

    from paper_2605_05099_b200 import shard

    r = state_io.create("x256**", seed=[1])
    fp = shard._fp([0.0, 1.0])
    ip = shard._ip([])
    info = _lib.RsRangeInfo()

    def call(rng, dist, entry, L, T):
        return _lib.lib.rs_range_count(ctypes.byref(rng.to_stream()), _lib.DIST_IDS[dist], fp, ip, entry, L, T,
                                       ctypes.byref(info), None)

    assert call(r, "norm", 0, 100, 256) == _lib.RS_ERR_VALUE      # seg_len not a multiple of 72
    assert call(r, "norm", 0, 144, 100) == _lib.RS_ERR_VALUE      # n_seg not a multiple of 256
    assert call(r, "norm", 144, 144, 256) == _lib.RS_ERR_VALUE    # entry beyond the first segment
    assert call(r, "u01", 0, 144, 256) == _lib.RS_ERR_UNSUPPORTED  # fixed consumption shards by offsets
    r.next_u64()                                                   # buffered words: not a fresh position
    assert call(r, "norm", 0, 144, 256) == _lib.RS_ERR_VALUE
    assert "fresh" in _lib.last_error()
    s = state_io.create("sfc64", seed=[1])                          # no skip-ahead
    assert call(s, "norm", 0, 144, 256) == _lib.RS_ERR_UNSUPPORTED


REF_SRC = pathlib.Path("/root/reference/pkg/src")


@pytest.mark.skipif(not (REF_SRC / "randstream" / "zigtables.py").exists(),
                    reason="the reference is only in the build container")
def test_tables_header_matches_reference_zigtables():
    """csrc/rs_tables.h (used by the kernels AND the oracle) is exactly what
    tools/gen_tables.py renders from the reference's zigtables.py: a stale table
    cannot move the product and its checker together unnoticed."""
    import runpy
    import sys

    argv = sys.argv
    sys.argv = ["gen_tables.py", str(REF_SRC)]
    try:
        g = runpy.run_path(str(ROOT / "tools" / "gen_tables.py"), run_name="gen_tables")
    finally:
        sys.argv = argv
    text = (ROOT / "paper_2605_05099_b200" / "csrc" / "rs_tables.h").read_text()
    assert g["render"]() == text


def test_serial_engine_warning_text():
    """Engines without skip-ahead warn once when a large single-stream fill is requested
    (the fill itself needs a GPU; here only the bookkeeping)."""
    import warnings as W
    from paper_2605_05099_b200 import rng as R
    R._serial_warned.discard("sfc64")
    with W.catch_warnings(record=True) as got:
        W.simplefilter("always")
        R._warn_serial("sfc64")
        R._warn_serial("sfc64")
    assert len(got) == 1 and "fill_streams" in str(got[0].message)
    assert set(R._SERIAL_ENGINES) == {"sfc64", "sfc64simd", "cwg128"}


def test_bench_reference_arm_line():
    """`bench.py --impl reference` (the CPU arm the driver launches beside ours): the port on all
    host threads over the headline's full config, one JSON line with the contract's keys, no GPU."""
    import json
    import pathlib
    import subprocess
    import sys

    root = pathlib.Path(__file__).resolve().parents[1]
    p = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 1 and line["higher_is_better"] is True
    assert line["unit"] == "Gsamples/s" and line["value"] > 0 and line["vs_baseline"] is None
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["config"]["same_config"] is True and "philox" in line["config"]["workload"]
