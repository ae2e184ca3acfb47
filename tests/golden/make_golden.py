"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

Run here (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_golden.py
Each case stores the plain inputs (reference gen_sparse, as its testutil
make_inputs does, P/tests/testutil.hpp:43-78), the blocked operands the
reference packed, the reference CPU kernel's output and counters
(run_parallel, backend automatic) and the 64-bit dense oracle output.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

# (name, (N, C, K, H, W, R, S, O, P), V, sparsity, seed)
CASES = [
    ("c3x3_s1_v16", (3, 32, 48, 9, 11, 3, 3, 1, 1), 16, 0.5, 11),
    ("c3x3_s2_v16", (2, 32, 32, 14, 13, 3, 3, 2, 2), 16, 0.6, 12),
    ("c1x1_s1_v16", (5, 48, 32, 7, 6, 1, 1, 1, 1), 16, 0.7, 13),
    ("c1x1_s2_v8", (2, 16, 16, 7, 7, 1, 1, 2, 2), 8, 0.4, 14),
    ("c5x5_s1_v4", (3, 8, 12, 8, 9, 5, 5, 1, 1), 4, 0.3, 15),
    ("c3x3_s1_v8_ragged", (19, 16, 24, 6, 7, 3, 3, 1, 1), 8, 0.8, 16),
    ("c3x3_s2_v4_full", (4, 8, 8, 5, 5, 3, 3, 2, 2), 4, 1.0, 17),
    ("c3x3_s1_v16_dense0", (2, 16, 16, 5, 5, 3, 3, 1, 1), 16, 0.0, 18),
]

COMPS = [(0, 0, "fwd"), (1, 0, "bwi"), (2, 0, "bww_in"), (2, 1, "bww_og")]


def make_inputs(sh, comp, check, s, seed):
    N, C, K, H, W, R, S = sh[:7]
    hp, wp = oracle.out_hw(sh)
    if comp == 0:
        return oracle.ref_gen_sparse(N, C, H, W, s, seed), oracle.ref_gen_sparse(K, C, S, R, 0.0, seed + 1)
    if comp == 1:
        return oracle.ref_gen_sparse(N, K, hp, wp, s, seed), oracle.ref_gen_sparse(K, C, S, R, 0.0, seed + 1)
    if check == 0:
        return oracle.ref_gen_sparse(N, C, H, W, s, seed), oracle.ref_gen_sparse(N, K, hp, wp, 0.0, seed + 2)
    return oracle.ref_gen_sparse(N, C, H, W, 0.0, seed), oracle.ref_gen_sparse(N, K, hp, wp, s, seed + 2)


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle ref)"
    for name, dims, V, s, seed in CASES:
        sh = oracle.ref_shape_make(*dims)
        blob = {"shape": np.array(sh, np.int32), "V": np.int32(V), "sparsity": np.float64(s)}
        for comp, check, tag in COMPS:
            a, b = make_inputs(sh, comp, check, s, seed)
            r = oracle.RefRun(comp, check, sh, V, a, b)
            out = {}
            for mode in (0, 1):
                r.exec(mode, 4)
                o, cnt, backend = r.result()
                out[mode] = (o, cnt)
            dense = oracle.ref_dense(comp, sh, a, b)
            blob[f"{tag}_a"] = a
            blob[f"{tag}_b"] = b
            blob[f"{tag}_a_blk"] = r.operand(0)
            blob[f"{tag}_b_blk"] = r.operand(1)
            blob[f"{tag}_ref_sparse"] = out[0][0]
            blob[f"{tag}_ref_dense_mode"] = out[1][0]
            blob[f"{tag}_oracle64"] = dense
            blob[f"{tag}_counters_sparse"] = np.array([out[0][1][k] for k in (
                "checked_vectors", "executed_vector_fmas", "output_vector_loads", "output_vector_stores")],
                np.uint64)
            blob[f"{tag}_counters_dense"] = np.array([out[1][1][k] for k in (
                "checked_vectors", "executed_vector_fmas", "output_vector_loads", "output_vector_stores")],
                np.uint64)
            r.close()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **blob)
        print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
