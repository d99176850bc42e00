"""Repeat decodes of a config many times; every result must equal the first (hang / race detector)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2406_06220_b200.decoder import LabelLoopingDecoder, Model
cfg = sys.argv[1] if len(sys.argv) > 1 else "fc-rnnt"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
spec, w, enc, lengths = bench.workload(cfg, 1000, sys.argv[3] if len(sys.argv) > 3 else "planted")
model = Model(w, spec.pred_kind, spec.context, spec.blank_id, spec.durations, "bf16")
dec = LabelLoopingDecoder(model, spec.max_symbols, enc.shape[0], enc.shape[1])
e = torch.from_numpy(enc).to("cuda", torch.bfloat16); l = torch.from_numpy(lengths).cuda()
print("setup done", flush=True)
out = dec.decode(e, l); ref = (out.tokens.clone(), out.lengths.clone())
print("first decode done", flush=True)
t0 = time.time()
for i in range(n):
    out = dec.decode(e, l)
    assert torch.equal(out.tokens, ref[0]) and torch.equal(out.lengths, ref[1]), f"mismatch at {i}"
    if i % 50 == 0:
        print("iter", i, flush=True)
print(cfg, "ok", n, "decodes", f"{(time.time()-t0)/n*1e3:.2f} ms each", flush=True)
