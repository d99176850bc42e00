import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import synth
from gpu_helpers import gpu_decode
from oracle import Transducer, decode_sequential
from oracle.verify import verify_rnnt

c = synth.CONFIGS["stateless-b512"]
spec = c["spec"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else c["B"]
w, enc, lengths, planted = synth.make_planted_rnnt(spec, 9, B, c["T_max"], c["len_lo"], c["len_hi"])
hyps, dec = gpu_decode(spec, w, enc, lengths, "bf16")
print("stats", dec.stats())
bad = [b for b in range(B) if (hyps[b][0], hyps[b][1]) != (planted[b][0], planted[b][1])]
print("mismatch rows", len(bad), bad[:20])
om = Transducer.from_spec(spec, w)
for b in bad[:3]:
    h, p = hyps[b], planted[b]
    n = min(len(h[0]), len(p[0]))
    i = next((k for k in range(n) if h[0][k] != p[0][k] or h[1][k] != p[1][k]), n)
    print(f"row {b} L={lengths[b]} gpu_len={len(h[0])} planted_len={len(p[0])} first diff @{i}: "
          f"gpu {h[0][i:i+3]} {h[1][i:i+3]} planted {p[0][i:i+3]} {p[1][i:i+3]}")
    r = verify_rnnt(om, enc[b], int(lengths[b]), spec.max_symbols, h[0], h[1])
    print("  verify gpu:", r.ok, r.message)
    o = decode_sequential(om, enc[b], int(lengths[b]), spec.max_symbols)
    print("  oracle == planted:", (o.tokens, o.timestamps) == (p[0], p[1]), " oracle == gpu:", (o.tokens, o.timestamps) == (h[0], h[1]))
