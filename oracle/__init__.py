"""CPU oracle for SVDQuant's W4A4 + low-rank linear (arXiv 2411.05007).

TEST INFRASTRUCTURE ONLY.  This package is the plain, slow, obviously-correct
reference that the CUDA path is checked against.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2411_05007_b200``) never imports it and shares no code with it.

Citations: ``P:n`` = PAPER.md line n (the LaTeX of the paper), ``S:n`` =
SPEC.md line n, ``§8(c)`` / ``App. B`` = SURVEY.md sections whose readings
are restated in DESIGN.md "Readings".

Modules
-------
formats      E2M1 / E4M3 / bf16 / fp16 codecs, nibble packing, 128x4 SF layout
quant        Eq. (1) quantizers: NVFP4 (g16, E4M3 scales) and INT4 (g64, 16-bit)
gptq         GPTQ quantization of the residual (App. D)
svdquant     smoothing, SVD split (Eq. 5), operand preparation, forward, LoRA
linalg       one-sided Jacobi SVD for tiny shapes (independent of LAPACK)
diagnostics  Eq. (3) error, Prop. 4.1 / 4.2 checks, cost fraction

Parity status of each function is listed in DESIGN.md ("Oracle pins").
Parity unpinned: the individual factors L1, L2 (sign / rotation freedom,
reading Q2) -- only their product and R are compared.
"""

from . import formats, quant, gptq, svdquant, linalg, diagnostics  # noqa: F401
