"""Time the fc-rnnt / fc-tdt decode under several (R, W, ring) configurations (ll_options overrides)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2406_06220_b200.decoder import LabelLoopingDecoder, Model
cfg = sys.argv[1] if len(sys.argv) > 1 else "fc-rnnt"
spec, w, enc, lengths = bench.workload(cfg, 1000)
model = Model(w, spec.pred_kind, spec.context, spec.blank_id, spec.durations, "bf16")
dec = LabelLoopingDecoder(model, spec.max_symbols, enc.shape[0], enc.shape[1])
e = torch.from_numpy(enc).to("cuda", torch.bfloat16); l = torch.from_numpy(lengths).cuda()
ref = None
from paper_2406_06220_b200 import ll
PAIRS = [tuple(map(int, x.split("x"))) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [(4, 8), (5, 6), (5, 4), (4, 4), (5, 2), (8, 4), (11, 2), (16, 2), (5, 1)]
for R, W in PAIRS:
    NS = 0
    ll.ll_set_options(ll.options(group_rows=R, window=W).opts)
    try:
        for _ in range(2):
            out = dec.decode(e, l)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); dec.launch(e, l); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
        st = dec.stats()
        h = (dec.tokens.clone(), dec.lengths_out.clone())
        same = ref is None or (torch.equal(h[0], ref[0]) and torch.equal(h[1], ref[1]))
        ref = ref or h
        print(f"R={R:2d} W={W} NS={NS or 'auto'} ms={np.median(ts):.3f} rounds/grp={st['joint_rounds']/st['groups']:.0f} "
              f"groups={st['groups']} same={same}", flush=True)
    except Exception as ex:
        print(f"R={R} W={W}: {ex}", flush=True)
