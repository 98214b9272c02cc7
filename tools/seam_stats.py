import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests'); sys.path.insert(0,'tests/golden')
import numpy as np, torch
import test_model_seam_gpu as T
import paper_2506_07900_b200 as P
b, sp, z = T._bundle()
for backend in ("dense","sparse"):
    sc = P.SparseAttentionConfig(**sp) if backend=="sparse" else None
    got = T._run(b, backend, sc, z["tokens"]); want = z[f"logits_{backend}"]
    e = np.abs(got-want); rowmax = e.max(1); scale = np.abs(want).max()
    print(backend, "scale", scale, "max", e.max(), "mean", e.mean(), "p50 row", np.median(rowmax), "p95 row", np.percentile(rowmax,95), "argmax agree", (got.argmax(-1)==want.argmax(-1)).mean(), "rows>0.05*scale", (rowmax>0.05*scale).sum())
