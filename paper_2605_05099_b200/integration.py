"""Route the reference's own front ends through the B200 fill path.

`install()` replaces `randstream.rng.Rng.fill` and `Rng.mvn` in an imported reference
package, so every caller of those methods -- the HTTP service's `/rngs/{h}/sample`
(pkg/src/randstream/service/app.py:148-162), the CLI `gen` (cli.py:83-125, which drives the
service in process), user code -- runs its bulk draws on the GPU with no other change:

    import randstream
    from paper_2605_05099_b200 import integration
    integration.install(randstream)

Each call adopts the reference generator's logical position (engine words, 144-word
buffer, pending half, mode flags, tallies; buffer.py:12-68), fills through `rs_fill` /
`rs_mvn_apply` with this package's `Rng` (same validation and messages as the reference,
rng.py:223-241, continuous.py:413-431), and writes the advanced position back into the
reference object, exactly as its own loop would have left it: later scalar draws,
`duplicate()` and checkpoints continue bit-for-bit. Results come back in the reference's
types (lists of Python ints / floats; an ndarray for `mvn`). Draws the device path does not
cover (`perm`, `sample`, fills below `min_n`) stay on the original methods.
"""

import functools

from . import engines
from .rng import DISCRETE_NAMES, SCALAR_NAMES, Rng

_DEVICE_DISTS = set(SCALAR_NAMES) | set(DISCRETE_NAMES)
_saved = {}


def adopt(ref_rng, device=None):
    """This package's Rng at the reference generator's exact logical position."""
    eid = engines.normalize(ref_rng.engine_id)
    ours = Rng(engines.make(eid))
    ours.engine.set_state([int(w) for w in ref_rng.engine.get_state()])
    ours.buffer.restore(ref_rng.buffer.capture())
    ours.bitexact = bool(ref_rng.bitexact)
    ours.full_mantissa = bool(ref_rng.full_mantissa)
    ours.counters = {k: dict(v) for k, v in ref_rng.counters.items()}
    ours.device = device
    return ours


def write_back(ours, ref_rng):
    """The advanced position (and tallies) back into the reference generator."""
    ref_rng.engine.set_state(list(ours.engine.get_state()))
    ref_rng.buffer.restore(ours.buffer.capture())
    ref_rng.counters = {k: dict(v) for k, v in ours.counters.items()}


def device_fill(ref_rng, dist, params=None, n=1, device=None):
    """`ref_rng.fill(dist, params, n)` computed on the GPU; the reference's list type."""
    ours = adopt(ref_rng, device)
    out = ours.fill(dist, params, n)  # validation errors raise before any state change
    write_back(ours, ref_rng)
    return out.cpu().tolist()


def device_mvn(ref_rng, mean, cov, n=1, layout="n_d", device=None):
    """`ref_rng.mvn(mean, cov, n, layout)` on the GPU (continuous.py:312-336)."""
    ours = adopt(ref_rng, device)
    out = ours.mvn(mean, cov, n=n, layout=layout)
    write_back(ours, ref_rng)
    return out.cpu().numpy()


def install(randstream=None, min_n=64, device=None):
    """Patch `randstream.rng.Rng.fill` / `.mvn` to run on the B200 path (idempotent).

    `min_n`: fills of fewer samples keep the reference's own loop (a device round trip
    costs more than a handful of Python draws)."""
    if randstream is None:
        import randstream  # noqa: F811
    R = randstream.rng.Rng
    if R in _saved:
        return
    orig_fill, orig_mvn = R.fill, R.mvn
    _saved[R] = (orig_fill, orig_mvn)

    def _slot(self, fn):
        # the reference's per-instance error slot (rng.py:38-52): success clears, failure records
        try:
            result = fn()
        except Exception as exc:
            self.last_error = str(exc) or type(exc).__name__
            raise
        self.last_error = None
        return result

    @functools.wraps(orig_fill)
    def fill(self, dist, params=None, n=1):
        if dist not in _DEVICE_DISTS or int(n) < min_n:
            return orig_fill(self, dist, params, n)
        return _slot(self, lambda: device_fill(self, dist, dict(params or {}), n, device))

    @functools.wraps(orig_mvn)
    def mvn(self, mean, cov, n=1, layout="n_d"):
        return _slot(self, lambda: device_mvn(self, mean, cov, n, layout, device))

    R.fill, R.mvn = fill, mvn


def uninstall(randstream=None):
    if randstream is None:
        import randstream  # noqa: F811
    R = randstream.rng.Rng
    if R in _saved:
        R.fill, R.mvn = _saved.pop(R)
