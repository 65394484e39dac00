"""Synthetic workloads of BASELINE.json (inputs are scalars: N, n or rho, seed).

No method arithmetic here: this module only names the configurations that
both the tests and bench.py use.
"""

# configs[0]: n=2^20 sorted without replacement from N=2^30, seed=1 (oracle in seconds)
CFG0 = dict(name="cfg0_wor_n2^20_N2^30", mode="wor", N=2 ** 30, n=2 ** 20, seed=1)
# configs[1]: n=2^30 from N=2^40, 1 B200 (single-GPU HBM-roofline run)
CFG1 = dict(name="cfg1_wor_n2^30_N2^40", mode="wor", N=2 ** 40, n=2 ** 30, seed=1)
# north_star headline: n=2^32 of N=2^48 on one GPU
HEADLINE = dict(name="wor_n2^32_N2^48", mode="wor", N=2 ** 48, n=2 ** 32, seed=1)
# configs[2]: weak scaling, n=2^30 per GPU from N=2^48
WEAK = dict(name="weak_wor_n2^30perGPU_N2^48", mode="wor", N=2 ** 48, n_per_gpu=2 ** 30, seed=1)
# configs[3]: dense n=0.75 N with N=2^32 (complement) and Bernoulli rho=0.01
CFG3A = dict(name="cfg3a_complement_n0.75N_N2^32", mode="wor", N=2 ** 32, n=3 * 2 ** 30, seed=1)
CFG3B = dict(name="cfg3b_bernoulli_rho0.01_N2^32", mode="bernoulli", N=2 ** 32, rho=0.01, seed=1)
CFG3B_ROOF = dict(name="bernoulli_rho0.01_N2^38", mode="bernoulli", N=2 ** 38, rho=0.01, seed=1)
# configs[4]: with replacement n=2^32 from N=2^36 (8 B200: 2^29 per GPU)
CFG4 = dict(name="cfg4_wr_n2^32_N2^36", mode="wr", N=2 ** 36, n=2 ** 32, seed=1)

# NEXT-3: G(V, m) with the edge decode fused into the leaf stores
GNM = dict(name="gnm_V2^23_m2^32", mode="gnm", V=2 ** 23, N=2 ** 22 * (2 ** 23 - 1), n=2 ** 32, seed=1)

# NEXT-4: Algorithm B + repair on the headline shape
ALGB = dict(name="algb_wor_n2^32_N2^48", mode="algb", N=2 ** 48, n=2 ** 32, seed=1, slack=4.0)

ALL = [CFG0, CFG1, HEADLINE, CFG3A, CFG3B, CFG3B_ROOF, CFG4]
PARITY_SEEDS = [0, 1, 0xDEADBEEF, 2 ** 64 - 1]


def paper_sweep():
    """Fig. 4's protocol: N = 2^50, n = 2^10..2^32, reps 2^30/n."""
    return [dict(name=f"sweep_n2^{e}_N2^50", mode="wor", N=2 ** 50, n=2 ** e, seed=1,
                 reps=max(1, 2 ** 30 // 2 ** e)) for e in range(10, 33, 2)]
