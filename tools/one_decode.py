"""One warm decode of a bench workload (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2406_06220_b200.decoder import LabelLoopingDecoder, Model
cfg = sys.argv[1] if len(sys.argv) > 1 else "fc-rnnt"
spec, w, enc, lengths = bench.workload(cfg, 1000)
model = Model(w, spec.pred_kind, spec.context, spec.blank_id, spec.durations, "bf16")
dec = LabelLoopingDecoder(model, spec.max_symbols, enc.shape[0], enc.shape[1])
e = torch.from_numpy(enc).to("cuda", torch.bfloat16); l = torch.from_numpy(lengths).cuda()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    dec.decode(e, l)
print(dec.stats())
