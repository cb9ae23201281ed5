"""Debug: the pull records against a numpy construction from the forward CSR."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import graphgen  # noqa
import paper_2311_10201_b200 as bpt  # noqa
from paper_2311_10201_b200 import bpt as B  # noqa
import torch
torch.cuda.set_device(0)
for name, scale in (("C1", 0), ("C2", 1 << 15)):
    cfg = graphgen.CONFIGS[name] if not scale else graphgen.scaled(graphgen.CONFIGS[name], scale, theta=64)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    m = len(col)
    out = np.zeros((m, 4), dtype=np.uint32)
    B._lib.bpt_debug_pull_records.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    rc = B._lib.bpt_debug_pull_records(g._h, out.ctypes.data)
    src = np.repeat(np.arange(len(row_ptr) - 1), np.diff(row_ptr.astype(np.int64)))
    order = np.lexsort((np.arange(m), col))  # stable by destination: reverse CSR position -> forward index
    e_of = np.empty(m, np.int64); e_of[order] = np.arange(m)
    # expected: grouped by u, inside a group by e
    exp = np.stack([src, col, e_of, thr], 1).astype(np.uint32)
    exp = exp[np.lexsort((exp[:, 2], exp[:, 0]))]
    print(name, "rc", rc, "equal", np.array_equal(out, exp), "rows differing", int((out != exp).any(1).sum()))
    bad = np.nonzero((out != exp).any(1))[0][:5]
    for i in bad: print("  ", i, out[i].tolist(), exp[i].tolist())
