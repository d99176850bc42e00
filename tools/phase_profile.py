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
ws = dec.workspace[off + 256: off + 256 + 25 * 8].cpu().numpy().view(np.uint64)
names = ["wait_f+plan", "build_z", "sync+spec issue", "joint", "exchange send", "exchange wait",
         "resolve", "sync", "decide", "sync+reload", "predictor", "outer/append", "", "", "", "TOTAL"]
tot = float(ws[15])
print(cfg, st)
rounds = st['joint_rounds'] / st['groups']
outer = st['outer_steps'] / st['groups']
print(f"per group: rounds {rounds:.1f}  outer steps {outer:.1f}  total cycles {int(tot)}")
for i, n in enumerate(names):
    if not n:
        continue
    v = ws[i]
    per = outer if i in (10, 11) else rounds
    print(f"{n:16s} {int(v):>10d} cycles  {100*v/tot:5.1f}%  per-{'step ' if i in (10, 11) else 'round'} {v/max(1, per):8.0f}")
sub = ["E'/setup", "gate MMA+wait", "gate epilogue", "sync", "h' exchange", "pred tiles", "sync2", "g exchange"]
npred = max(1, st['predictor_steps'] / st['groups'])
for i, nm in enumerate(sub):
    print(f"  pred.{nm:16s} {ws[16+i]/npred:9.0f} cycles/step")
