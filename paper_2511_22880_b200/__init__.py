"""paper_2511_22880_b200 — B200-native mixed-rank LoRA delta path of LoRAServe (arxiv 2511.22880).

Host side mirrors the reference's Python API for the path (costmodel / placement / routing /
pool / domain / demand / traces) and drives liblsv, a C-ABI library of hand-written sm_100a
kernels (include/lsv.h).  See DESIGN.md.
"""

__version__ = "0.1.0"
