"""The reference's own HTTP service (`/rngs/{h}/sample`, pkg/src/randstream/service/app.py:
148-162) driven through `integration.install()`.

Runs in the build container, where the reference is importable and there is no GPU: the
device fill under the hook is replaced by a stand-in computed by the oracle at the same
logical position (the test checks the hook's hand-off -- adopting the reference
generator's engine words, buffer, pending half and flags, writing the advanced position
back -- not the kernels, which the GPU parity tests cover). Every response and every later
draw must equal the unhooked reference service's."""
import pathlib
import sys

import numpy as np
import pytest
import torch

REF = pathlib.Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not (REF / "randstream" / "service" / "app.py").exists(),
                                reason="the reference is only in the build container")


def _oracle_at(rng):
    from oracle import oracle as O
    o = O.OracleRng(rng.engine_id)
    st = rng.engine.get_state()
    for i, w in enumerate(st):
        o.r.st[i] = w
    cap = rng.buffer.capture()
    for i, w in enumerate(cap["words"]):
        o.r.buf[i] = w
    o.r.fill, o.r.cursor = cap["fill"], cap["cursor"]
    o.r.has_pending = int(cap["pending"] is not None)
    o.r.pending = cap["pending"] or 0
    o.r.full_mantissa = int(rng.full_mantissa)
    return o


def _stand_in_fill(self, dist, params=None, n=1, out=None):
    """The device fill's contract (values + post-fill position + tallies), on the oracle,
    after the product's own parameter validation (rng.py _continuous_params / _discrete_params)."""
    from paper_2605_05099_b200.rng import DISCRETE_NAMES
    params = dict(params or {})
    if dist in DISCRETE_NAMES:
        self._discrete_params(dist, params, n)
    else:
        self._continuous_params(dist, params, n)
    o = _oracle_at(self)
    vals = o.fill(dist, dict(params or {}), n)
    self.engine.s = o.get_state()
    words, cursor, pending = o.buffer()
    self.buffer.restore({"capacity": 144, "fill": len(words), "cursor": cursor, "words": words,
                         "pending": pending})
    for name, t in o.tallies().items():
        c = self.counters.setdefault(name, {"attempts": 0, "pdf_evals": 0})
        c["attempts"] += t["attempts"]
        c["pdf_evals"] += t["pdf_evals"]
    return torch.from_numpy(vals)


def _stand_in_mvn(self, mean, cov, n=1, layout="n_d"):
    """rs_mvn_apply's contract on the host: z from the stand-in fill, X = mean + z @ L^T."""
    from paper_2605_05099_b200.rng import semidefinite_factor
    mean = np.asarray(mean, dtype=np.float64)
    L = semidefinite_factor(np.asarray(cov, dtype=np.float64))
    o = _oracle_at(self)
    z = o.fill("stdnorm", {}, n * mean.size).reshape(n, mean.size)
    self.engine.s = o.get_state()
    words, cursor, pending = o.buffer()
    self.buffer.restore({"capacity": 144, "fill": len(words), "cursor": cursor, "words": words,
                         "pending": pending})
    x = mean + z @ L.T
    return torch.from_numpy(x if layout == "n_d" else np.ascontiguousarray(x.T))


@pytest.fixture()
def apps(monkeypatch):
    sys.path.insert(0, str(REF))
    import randstream
    from fastapi.testclient import TestClient
    from randstream.service.app import create_app

    from paper_2605_05099_b200 import integration
    from paper_2605_05099_b200.rng import Rng

    plain = TestClient(create_app())
    monkeypatch.setattr(Rng, "fill", _stand_in_fill)
    monkeypatch.setattr(Rng, "mvn", _stand_in_mvn)
    integration.install(randstream, min_n=64)
    try:
        yield plain, TestClient(create_app()), randstream
    finally:
        integration.uninstall(randstream)


def _make(client, engine, seed):
    r = client.post("/rngs", json={"engine": engine, "seed": [str(s) for s in seed]})
    assert r.status_code == 201, r.text
    return r.json()["handle"]


def _sample(client, h, dist, params, n):
    r = client.post("/rngs/%s/sample" % h, json={"dist": dist, "params": params, "n": n})
    assert r.status_code == 200, r.text
    return r.json()["values"]


CASES = [("x256**", "norm", {}), ("pcg64", "gamma", {"alpha": 2.5}), ("philox", "u01f", {}),
         ("ranlux++", "uint64", {}), ("sfc64", "uint64", {"b": "1000003"}), ("pcg64", "beta", {"a": 2.0, "b": 5.0}),
         ("x256++simd", "exp", {"beta": 2.0}), ("philox", "normf", {}), ("x256**", "int", {"m": -5, "n": 17})]


@pytest.mark.parametrize("engine,dist,params", CASES)
def test_service_sample_through_the_hook(apps, engine, dist, params):
    plain, hooked, randstream = apps
    # the reference's own route: sample values are strings for uint64 (app.py:20-21, 160-161)
    p = {k: (int(v) if isinstance(v, str) else v) for k, v in params.items()}
    hp, hh = _make(plain, engine, [2024]), _make(hooked, engine, [2024])
    # a small draw first (below min_n: the reference loop) leaves the stream mid-buffer
    assert _sample(plain, hp, "u01f", {}, 3) == _sample(hooked, hh, "u01f", {}, 3)
    for n in (1000, 4097):
        assert _sample(plain, hp, dist, p, n) == _sample(hooked, hh, dist, p, n), (dist, n)
    # the stream continues identically after the device fill: scalar draws, state, checkpoint
    assert _sample(plain, hp, "uint64", {}, 5) == _sample(hooked, hh, "uint64", {}, 5)
    assert plain.get("/rngs/%s/state" % hp).json() == hooked.get("/rngs/%s/state" % hh).json()
    assert plain.get("/rngs/%s/serialized" % hp).json() == hooked.get("/rngs/%s/serialized" % hh).json()


def test_mvn_and_fallbacks_through_the_hook(apps):
    plain, hooked, randstream = apps
    # perm / sample draws and small fills stay on the reference loop (nothing to route)
    hp, hh = _make(plain, "x256**", [7]), _make(hooked, "x256**", [7])
    for dist, params, n in (("perm", {"n": 20}, 1), ("norm", {}, 10)):
        r1 = plain.post("/rngs/%s/sample" % hp, json={"dist": dist, "params": params, "n": n})
        r2 = hooked.post("/rngs/%s/sample" % hh, json={"dist": dist, "params": params, "n": n})
        assert r1.status_code == r2.status_code and r1.json() == r2.json()
    # an invalid request fails the same way through the hook, and leaves the stream alone
    bad = {"dist": "gamma", "params": {"alpha": -1.0}, "n": 500}
    r1 = plain.post("/rngs/%s/sample" % hp, json=bad)
    r2 = hooked.post("/rngs/%s/sample" % hh, json=bad)
    assert r1.status_code == r2.status_code != 200 and r1.json() == r2.json()
    assert plain.get("/rngs/%s/error" % hp).json() == hooked.get("/rngs/%s/error" % hh).json()
    assert plain.get("/rngs/%s/state" % hp).json() == hooked.get("/rngs/%s/state" % hh).json()
    # mvn through the hook: the reference's mean + z @ L^T on the same z stream
    req = {"dist": "mvn", "params": {"mean": [0.5, -1.0, 2.0], "cov": [[2.0, 0.3, 0.1], [0.3, 1.0, 0.2],
                                                                       [0.1, 0.2, 1.5]]}, "n": 300}
    x1 = np.array(plain.post("/rngs/%s/sample" % hp, json=req).json()["values"])
    x2 = np.array(hooked.post("/rngs/%s/sample" % hh, json=req).json()["values"])
    assert x1.shape == x2.shape == (300, 3)
    assert np.max(np.abs(x1 - x2)) <= 1e-12 * np.max(np.abs(x1))
    assert plain.get("/rngs/%s/state" % hp).json() == hooked.get("/rngs/%s/state" % hh).json()


def test_install_is_idempotent_and_reversible():
    sys.path.insert(0, str(REF))
    import randstream

    from paper_2605_05099_b200 import integration
    orig = randstream.rng.Rng.fill
    integration.install(randstream)
    patched = randstream.rng.Rng.fill
    integration.install(randstream)
    assert randstream.rng.Rng.fill is patched and patched is not orig
    integration.uninstall(randstream)
    assert randstream.rng.Rng.fill is orig
