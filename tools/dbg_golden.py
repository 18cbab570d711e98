import sys, json, hashlib
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from paper_2605_05099_b200 import state_io
from conftest import golden_params, is_vectorized, vec_close
g = json.load(open("/root/repo/tests/golden/reference_vectors.json"))
arr = np.load("/root/repo/tests/golden/reference_arrays.npz")
bad = []
for rec in g["fills"]:
    r = state_io.create(rec["engine"], seed=rec["seed"], spawn_key=tuple(rec["spawn"]))
    r.set_full_mantissa(rec["full_mantissa"]); r.set_bitexact(rec.get("bitexact", False))
    for op in rec["pre"]:
        for _ in range(op[1]): (r.next_u64 if op[0] == "u64" else r.next_u32)()
    try:
        out = r.fill(rec["dist"], golden_params(rec), rec["n"]).cpu().numpy()
    except Exception as e:
        bad.append((rec["name"], "EXC " + str(e))); continue
    ok = vec_close(out, arr[rec["name"]]) if is_vectorized(rec) else hashlib.sha256(np.ascontiguousarray(out).tobytes()).hexdigest() == rec["sha256"]
    if not ok:
        if rec["name"] in arr.files and not is_vectorized(rec):
            ref = arr[rec["name"]]; d = np.nonzero(out.view(np.uint8).reshape(len(out), -1).any(1) != ref.view(np.uint8).reshape(len(ref), -1).any(1))[0]
            w = np.nonzero(out.tobytes() != ref.tobytes())
        bad.append((rec["name"], "output"))
        continue
    cap = r.buffer.capture()
    st_ok = r.get_state() == [int(w, 16) for w in rec["final_state"]] and cap["cursor"] == rec["cursor"] and (None if cap["pending"] is None else "%08x" % cap["pending"]) == rec["pending"]
    if not st_ok: bad.append((rec["name"], "state"))
    elif r.counters != rec["tallies"]: bad.append((rec["name"], "tally %s vs %s" % (r.counters, rec["tallies"])))
print(len(bad), "bad")
for b in bad: print(b)
