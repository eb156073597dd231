"""DLIC CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of the DLIC hot path
(arXiv 2207.05152, /root/reference/PAPER.md cited as P:<line>), written from
the paper and the readings R1-R10 of SURVEY.md / DESIGN.md.  Every function
cites the passage it follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2207_05152_b200``) never imports it and shares no code
with it; the only shared module is ``synth`` (seeded inputs, no method
arithmetic).

Modules
-------
window    causal 9x9 window (Fig. 6), out-of-image fill 0
schedule  wavefront step(r, c) = c + 3r (P:87 WPP, Fig. 1 right)
mlp       dense density estimator, 6 layers, ReLU, 256 logits
quant     softmax and the Q1 PDF -> integer table (paper silent; R5)
rans      32-bit rANS coder (constants R6)
streams   per-row lanes interleaved into G-row group streams (R7)
container byte container (framing unstated)
model_io  "DLICMDL1" model file + SHA-256 content hash
codec     encode / wavefront decode / raster decode
train     brief trainer producing fixture weights

Parity pins for every function live in tests/test_oracle_*.py.  Functions
with no independent pin say "parity unpinned" in their docstring.
"""

from . import window, schedule, mlp, quant, rans, streams, container, model_io, codec  # noqa: F401
