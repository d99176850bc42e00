"""LSTM ring-path correctness for given dims (cluster size chosen by the library)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth
from gpu_helpers import gpu_decode
dt = sys.argv[1] if len(sys.argv) > 1 else "bf16"
dims = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "129,128,128,128").split(",")]
spec = synth.ModelSpec(dims[0], dims[1], dims[2], dims[3], "lstm", 1, None, 0, 10)
w, enc, lengths, planted = synth.make_planted_rnnt(spec, 5, 8, 60, 40, 60)
hyps, dec = gpu_decode(spec, w, enc, lengths, dt)
st = dec.stats()
bad = [b for b in range(8) if (hyps[b][0], hyps[b][1]) != tuple(planted[b][:2])]
print(f"C={st['cluster_size']} R={st['group_rows']} W={st['window']} dtype={dt} mismatching rows: {bad}")
if bad:
    b = bad[0]; h = hyps[b]; p = planted[b]
    n = min(len(h[0]), len(p[0]))
    i = next((k for k in range(n) if (h[0][k], h[1][k]) != (p[0][k], p[1][k])), n)
    print("  first diff @", i, "gpu", h[0][i:i+3], h[1][i:i+3], "planted", p[0][i:i+3], p[1][i:i+3])
