"""Per-phase clock64 profile of the decode kernel (cluster 0, rank 0, thread 0).
Run with LL_PROFILE=1 on a GPU box: python tools/phase_profile.py [config]"""
import os, sys
os.environ["LL_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2406_06220_b200.decoder import LabelLoopingDecoder, Model
cfg = sys.argv[1] if len(sys.argv) > 1 else "fc-rnnt"
spec, w, enc, lengths = bench.workload(cfg, 1000)
model = Model(w, spec.pred_kind, spec.context, spec.blank_id, spec.durations, "bf16")
dec = LabelLoopingDecoder(model, spec.max_symbols, enc.shape[0], enc.shape[1])
e = torch.from_numpy(enc).to("cuda", torch.bfloat16); l = torch.from_numpy(lengths).cuda()
for _ in range(3):
    dec.decode(e, l)
st = dec.stats()
off = dec.ws_ptr - dec.workspace.data_ptr()
ws = dec.workspace[off + 256: off + 256 + 17 * 8].cpu().numpy().view(np.uint64)
names = ["wait_f", "build_z", "joint", "exchange", "decide", "predictor", "outer/append", "TOTAL"]
tot = float(ws[7])
print(cfg, st)
rounds = st['joint_rounds'] / st['groups']
for n, v in zip(names, ws[:8]):
    print(f"{n:14s} {int(v):>12d} cycles  {100*v/tot:5.1f}%  per-round {v/max(1, rounds):8.0f}")
print("per predictor step:", ws[5] / max(1, st['predictor_steps'] / st['groups']))
sub = ["E'/setup", "gate MMA+wait", "gate epilogue", "sync", "h' exchange", "pred tiles", "sync2", "g exchange"]
npred = max(1, st['predictor_steps'] / st['groups'])
for i, nm in enumerate(sub):
    print(f"  pred.{nm:16s} {ws[8+i]/npred:9.0f} cycles/step")
print(f"  pred.tile-wait     {ws[16]/npred:9.0f} cycles/step (inside MMA)")
