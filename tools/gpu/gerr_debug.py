"""Debug: which g rows / dims of the production probe deviate from float64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np, torch
import synth
from gpu_helpers import gpu_model
from oracle import Transducer
from paper_2406_06220_b200.decoder import LabelLoopingDecoder, probe_decode
from test_gpu_parity import _oracle_g_sequence
spec = synth.ModelSpec(1025, 512, 640, 640, "lstm", 1, None, 0, 10)
w = synth.make_weights(spec, 61, blank_bias=synth.random_family_blank_bias(spec))
B, T = 16, 80
enc, lengths = synth.make_inputs(62, B, T, spec.enc_dim, 40, T)
model = gpu_model(spec, w)
dec = LabelLoopingDecoder(model, spec.max_symbols, B, T)
out, jrows, grows = probe_decode(dec, torch.from_numpy(enc).to("cuda", torch.bfloat16), torch.from_numpy(lengths).cuda())
hyps = out.hypotheses()
o = Transducer.from_spec(spec, w)
gseq = {b: _oracle_g_sequence(o, hyps[b][0]) for b in range(B)}
bad = []
for b, n, g in grows:
    e = np.abs(g.astype(np.float64) - gseq[b][n])
    if e.max() > 1e-3:
        dims = np.nonzero(e > 1e-3)[0]
        bad.append((b, n, e.max(), sorted(set(int(d) // 40 for d in dims)), len(dims)))
print("bad g rows:", len(bad), "of", len(grows))
for r in bad[:20]:
    print(r)
print(dec.stats())
