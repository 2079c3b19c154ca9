"""Layer compositions on top of the C ABI (argument marshalling only; every
step of the recurrence runs in libsrnn's kernels).

Bidirectional layer (SURVEY.md Sec. 8(f)4 "bidirectional cells"; the paper's
DS2 case study uses recurrent layers of a bidirectional speech model,
PAPER.md:318): a forward plan over x and a backward plan over x reversed in
time, outputs concatenated along the feature axis, y = [y_fwd ; flip(y_bwd)].
The two directions are independent recurrences, but they run one after the
other, each on all SMs: two persistent kernels on half of the SMs each, launched
on two streams, were measured 8-17x slower on B200 (``scripts/bidir_time.py``,
``profiles/r01_exchange_experiments.md``) -- spinning persistent kernels must
not share the GPU.
"""
from __future__ import annotations

from ._lib import SparseRNN, from_problem


class BiSparseRNN:
    def __init__(self, fwd: SparseRNN, bwd: SparseRNN):
        if (fwd.H, fwd.I, fwd.G) != (bwd.H, bwd.I, bwd.G):
            raise ValueError("both directions need the same hidden, input and cell")
        self.fwd, self.bwd = fwd, bwd
        self.H, self.I, self.G = fwd.H, fwd.I, fwd.G

    @classmethod
    def from_problems(cls, prob_f, prob_b, prec="fp16", device=0, flags=0, num_ctas=0):
        """Two plans from problem dicts (``inputs.make_problem``)."""
        return cls(from_problem(prob_f, prec=prec, device=device, flags=flags, num_ctas=num_ctas),
                   from_problem(prob_b, prec=prec, device=device, flags=flags, num_ctas=num_ctas))

    def forward(self, x, h0=None, streams=None):
        """x: [T, B, I] CUDA float32 -> (y [T, B, 2H], hT_fwd, hT_bwd).  h0: optional (h0_fwd, h0_bwd).
        streams: optional (s_fwd, s_bwd) for the two directions (experiments only, see module doc)."""
        import torch
        h0f, h0b = h0 if h0 is not None else (None, None)
        xr = torch.flip(x, dims=[0]).contiguous()
        if streams is not None:
            cur = torch.cuda.current_stream()
            s1, s2 = streams
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            with torch.cuda.stream(s1):
                of = self.fwd.forward(x, h0f, stream=s1)
            with torch.cuda.stream(s2):
                ob = self.bwd.forward(xr, h0b, stream=s2)
            cur.wait_stream(s1)
            cur.wait_stream(s2)
        else:
            of = self.fwd.forward(x, h0f)
            ob = self.bwd.forward(xr, h0b)
        y = torch.cat([of[0], torch.flip(ob[0], dims=[0])], dim=2)
        return y, of[1], ob[1]

    def status(self):
        self.fwd.status()
        self.bwd.status()

    def close(self):
        self.fwd.close()
        self.bwd.close()
