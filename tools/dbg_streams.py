import sys, subprocess
sys.path.insert(0, ".")
cases = [("x256**", "norm", {}, 96, 1), ("x256**", "norm", {}, 8, 1), ("x256**", "exp", {}, 96, 10), ("x256**", "u01", {}, 96, 10)]
if len(sys.argv) > 1:
    from paper_2605_05099_b200 import fill_streams
    eng, dist, params, S, n = cases[int(sys.argv[1])]
    out = fill_streams(eng, [7], [4], 5, S, dist, params, n)
    import torch; torch.cuda.synchronize()
    print("ok", out.shape)
else:
    for i, c in enumerate(cases):
        r = subprocess.run([sys.executable, __file__, str(i)], capture_output=True, text=True)
        print(c, r.stdout.strip()[-40:], r.stderr.strip().splitlines()[-1:] if r.returncode else "")
