import sys, numpy as np
sys.path.insert(0, '.')
import oracle as O, paper_2512_17910_b200 as P
def run(dims, use_ad, label):
    ocfg = O.OracleConfig(**dims, numerics="bf16"); om = O.OracleModel(ocfg)
    pm = P.Model(P.ModelConfig(**dims, dtype="bf16"))
    V = dims["vocab_size"]; inv = (V-32, V-31, V-30)
    rng = np.random.default_rng(0)
    toks = np.concatenate([rng.integers(0, V-32, 90), inv, rng.integers(0, V-32, 4)])
    ids = list(range(8)); mask = np.arange(len(toks)) < 90
    oa = O.oracle_adapter("a0", ocfg, 32, seed=2, invocation_tokens=inv) if use_ad else None
    pa = P.generate_adapter("a0", ocfg.d_model, 32, seed=2, invocation_tokens=inv, kv_width=ocfg.kv_width, q_width=ocfg.q_width) if use_ad else None
    okv = om.new_pool(8, 16); pool = P.BlockPool(8, 16, dims["n_layers"], ocfg.d_model, kv_width=ocfg.kv_width, dtype="bf16")
    w = om.forward_step([O.OracleSpan("r", toks, 0, ids, oa, mask if use_ad else None)], okv)["r"]
    g = pm.forward_step([P.SeqInput("r", toks, 0, ids, pa, mask if use_ad else None)], pool.kv)["r"]
    kv = pool.kv.float().cpu().numpy()
    print(f"{label:30s} |dlogit| {np.abs(g-w).max():.4f} scale {np.abs(w).max():.2f} kvrel {np.linalg.norm(kv-okv)/np.linalg.norm(okv):.4g} kvmax {np.abs(kv-okv).max():.4g}")
    # per layer kv error
    for l in range(dims["n_layers"]):
        print("   layer", l, "K rel", np.linalg.norm(kv[:,l,0]-okv[:,l,0])/np.linalg.norm(okv[:,l,0]), "V rel", np.linalg.norm(kv[:,l,1]-okv[:,l,1])/np.linalg.norm(okv[:,l,1]))
base = dict(arch="llama", n_layers=2, n_heads=8, n_kv_heads=2, head_dim=64, d_model=256, ffn_dim=512, vocab_size=320, seed=1)
run(base, False, "llama gqa no adapter")
run(base, True, "llama gqa activated")
run(dict(base, n_kv_heads=8), False, "llama mha")
run(dict(base, n_layers=1), False, "llama 1 layer")
C1 = dict(n_layers=2, n_heads=4, head_dim=64, d_model=256, vocab_size=256, seed=0)
run(C1, True, "ref c1 activated")
