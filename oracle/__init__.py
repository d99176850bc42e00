"""Float64 CPU oracle for label-looping greedy Transducer decoding.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import this package.
The product path (`paper_2406_06220_b200/`, `include/ll.h`, the CUDA library)
never imports, links or executes anything here, and this package imports
nothing from the product path: the two share no code.  Inputs come from
`synth/` (seeded generators with no method arithmetic).

Contents (each function cites the passage it follows, PAPER.md line numbers):
  model.py   -- the Transducer pieces in float64: encoder projection (Alg. 3
                line 2, §3.4), LSTM / stateless predictor (Alg. 1 lines 6-8,
                §1 contribution 3), predictor projection (§3.4), ReLU joint
                with optional TDT duration head (§2, §3.3).
  decode.py  -- Alg. 1 sequential greedy decoding (THE oracle definition) for
                RNN-T and TDT, Alg. 2 batched frame-looping, and Alg. 3
                batched label-looping (CPU reference of the GPU method), with
                the readings of DESIGN.md §"Readings".
  brute.py   -- brute-force enumeration of all well-formed alignments on tiny
                inputs (pin: unique greedy-consistent alignment).
  verify.py  -- teacher-forced verifier: replays a decoder's outputs through
                the float64 model and accepts a decision iff it is the
                float64 argmax or within the near-tie tolerance.

Pins (tests/test_oracle_*.py, `-m "not gpu"`): Fig. 2 CAT/DOG worked example,
closed forms (always-blank, never-blank guard, TDT forced alignment), brute
force, Alg.1 == Alg.2 == Alg.3 bit-exactness, torch.nn.LSTMCell / numpy
matmul special cases, planted-alignment closed form at full scale.
Parity status of every function is listed in DESIGN.md §"Oracle pins".
"""
from .model import Transducer, argmax_lowest  # noqa: F401
from .decode import (  # noqa: F401
    decode_sequential, decode_frame_looping, decode_label_looping, DecodeResult,
)
