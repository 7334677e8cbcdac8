"""Generate tests/golden/reference_vectors.npz from the UNMODIFIED reference.

Run here (where /root/reference is mounted and oracle/_ref is built):
    python tests/golden/make_golden.py
The fixtures pin the oracle restatement (tests/test_golden.py) on hosts where
the reference library cannot be built (e.g. the GPU box): every array below is
an output of the reference's own public functions (oracle/_ref/libedgekv_refc.so,
compiled from /root/reference/proj/src), on seeded inputs stored alongside.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Reference, build, model_from_reference_layout  # noqa: E402


def main():
    build(ref=True)
    ref = Reference()
    g = {}
    # rng.hpp: raw mt19937_64 + Rng::mix
    g["mt_seed"] = np.array([42], dtype=np.uint64)
    g["mt_stream"] = ref.mt64_stream(42, 64)
    g["mix_in"] = np.array([[0, 0], [42, 0x9B0BE], [12345, 7]], dtype=np.uint64)
    g["mix_out"] = np.array([ref.mix(int(a), int(b)) for a, b in g["mix_in"]], dtype=np.uint64)
    # transformer.cpp:82-115 init_model + checksum (golden fa0d3d12020757f7)
    m = ref.init_model(2, 2, 4, 32, 12345)
    g["model_checksum"] = np.array([m["checksum"]], dtype=np.uint64)
    for k in ("wq", "wk", "wv", "out_proj", "pos"):
        g["model_" + k] = m[k]
    g["embeddings"] = ref.generate_embeddings(99, 5, 12)
    # head_prune.cpp: from_lambda budgets and select_channels
    lam = [(0.2, 80), (0.0, 7), (1.0, 7), (1 / 3, 6), (0.5, 7), (0.5, 128), (0.25, 64)]
    g["from_lambda_in"] = np.array(lam)
    g["from_lambda_out"] = np.array([ref.prune_retained(a, int(b)) for a, b in lam])
    rng = np.random.default_rng(2026)
    scale = np.exp(rng.uniform(-1.5, 1.5, 16))
    g["sel_q"] = rng.uniform(-1, 1, (24, 16)) * scale
    g["sel_k"] = rng.uniform(-1, 1, (30, 16)) * scale[::-1]
    g["sel_kept"] = ref.select_channels(g["sel_q"], g["sel_k"], 0.5)
    g["prune_objective"] = np.array([ref.prune_objective(g["sel_q"], g["sel_k"], g["sel_kept"])])
    # cache_merge.cpp: segment attention + Eq. 5 merge
    g["seg_q"] = rng.uniform(-2, 2, 8)
    g["seg_k"] = rng.uniform(-2, 2, (11, 8))
    g["seg_v"] = rng.uniform(-2, 2, (11, 8))
    c = ref.segment_attention(g["seg_q"], g["seg_k"][:6], g["seg_v"][:6])
    u = ref.segment_attention(g["seg_q"], g["seg_k"][6:], g["seg_v"][6:])
    g["seg_ctx"] = np.concatenate([c[0], [c[1], c[2]]])
    g["seg_user"] = np.concatenate([u[0], [u[1], u[2]]])
    mo = ref.merge_attention(c, u)
    g["merge_out"] = np.concatenate([mo[0], [mo[1], mo[2]]])
    # collaborative_decode on the golden model with a context from its own prefill
    L, H, d, mp = 2, 2, 4, 32
    model = model_from_reference_layout(m, L, H, d, mp)
    ctx_emb = ref.generate_embeddings(41, 5, 8)
    _, ck, cv = ref.prefill(model, ctx_emb)
    user = ref.generate_embeddings(43, 3, 8)
    pre, steps = ref.collaborative_decode(model, ck, cv, user, 4, boundary=1)
    g["cd_ctx_emb"], g["cd_user"], g["cd_prefill"], g["cd_steps"] = ctx_emb, user, pre, steps
    # layer_match.cpp: match_layers on two init_model models
    e = model_from_reference_layout(ref.init_model(3, 2, 6, 64, 41), 3, 2, 6, 64)
    cl = model_from_reference_layout(ref.init_model(5, 4, 6, 64, 43), 5, 4, 6, 64)
    eo = ref.prefill(e, ref.generate_embeddings(9, 16, 12))[0]
    co = ref.prefill(cl, ref.generate_embeddings(9, 16, 24))[0]
    cka, rsa, best = ref.match_layers(eo, co, 0.5, 0.3)
    g["ml_edge"], g["ml_cloud"], g["ml_cka"], g["ml_rsa"], g["ml_best"] = eo, co, cka, rsa, best
    # cost_model.cpp: cache_source + pipeline_schedule
    cs = [(5, 0.1, 99.0, 4, 6), (6, 0.0, 0.0, 4, 6), (2, 1.0, 2.0, 4, 6), (2, 3.0, 2.0, 4, 6),
          (1, 2.0, 2.0, 4, 6)]
    g["cs_in"] = np.array(cs)
    g["cs_out"] = np.array([ref.cache_source(*c_) for c_ in cs])
    tcomm = rng.uniform(0, 10, 9)
    tcomp = rng.uniform(0, 10, 9)
    pip, seq, tot = ref.pipeline_schedule(tcomm, tcomp)
    g["ps_comm"], g["ps_comp"], g["ps_pip"] = tcomm, tcomp, pip
    g["ps_tot"] = np.array([seq, tot])
    out = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(out, **g)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
