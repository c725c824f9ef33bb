"""Generate the golden fixtures by running the REFERENCE itself (omnisim 0.1.0).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

The GPU box never reads /root/reference; it only sees the committed .npz files.
Every fixture records the exact reference call that produced it.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    import omnisim as om  # noqa: E402  (the reference)

    rng = np.random.default_rng(20261018)

    # 1. lowering, bit-exact targets (tensors.lower, tensors.py:164-181)
    lower_cases = [(2, 3, 9, 3, 1, 1), (3, 1, 8, 3, 1, 1), (2, 3, 27, 11, 4, 0), (1, 5, 13, 5, 2, 2),
                   (4, 2, 6, 1, 1, 0), (2, 2, 7, 3, 2, 0)]
    arrs = {}
    for i, (b, c, n, k, s, p) in enumerate(lower_cases):
        D = rng.standard_normal((b, c, n, n)).astype(np.float32).astype(np.float64)
        spec = om.ConvSpec(n=n, k=k, d_in=c, d_out=1, stride=s, pad=p)
        start, b_p = (1, b - 1) if b > 1 else (0, 1)
        arrs[f"case{i}_geom"] = np.array([b, c, n, k, s, p, start, b_p])
        arrs[f"case{i}_D"] = D
        arrs[f"case{i}_Dhat"] = om.lower(om.Tensor4(D), spec, b_p=b_p, start=start).matrix
    np.savez_compressed(os.path.join(OUT, "lower.npz"), **arrs)

    # 2. conv_lowered / conv_direct / gemm / lift (tensors.py:144-256) incl. SPEC KATs
    arrs = {}
    conv_cases = [(8, 3, 2, 4, 1, 0, 8), (9, 3, 3, 5, 2, 1, 3), (13, 5, 4, 6, 1, 2, 2),
                  (12, 4, 1, 3, 4, 0, 2), (6, 1, 2, 3, 1, 0, 4)]
    for i, (n, k, din, dout, s, p, b) in enumerate(conv_cases):
        spec = om.ConvSpec(n=n, k=k, d_in=din, d_out=dout, stride=s, pad=p)
        D = rng.standard_normal((b, din, n, n)).astype(np.float32).astype(np.float64)
        Kw = rng.standard_normal((dout, din, k, k)).astype(np.float32).astype(np.float64)
        arrs[f"conv{i}_geom"] = np.array([n, k, din, dout, s, p, b])
        arrs[f"conv{i}_D"] = D
        arrs[f"conv{i}_K"] = Kw
        arrs[f"conv{i}_R"] = om.conv_lowered(om.Tensor4(D), om.Tensor4(Kw), spec, b_p=b,
                                             workers=2).values
        arrs[f"conv{i}_Rdirect"] = om.conv_direct(om.Tensor4(D), om.Tensor4(Kw), spec).values
    # SPEC.md:49 KAT: 3x3 input 1..9, 2x2 kernel [[1,0],[0,1]] -> [[6,8],[12,14]]
    spec = om.ConvSpec(n=3, k=2, d_in=1, d_out=1)
    D = np.arange(1, 10, dtype=np.float64).reshape(1, 1, 3, 3)
    Kw = np.array([[1.0, 0.0], [0.0, 1.0]]).reshape(1, 1, 2, 2)
    arrs["kat_D"], arrs["kat_K"] = D, Kw
    arrs["kat_R"] = om.conv_lowered(om.Tensor4(D), om.Tensor4(Kw), spec).values
    A = rng.standard_normal((37, 300))
    B = rng.standard_normal((300, 11))
    arrs["gemm_A"], arrs["gemm_B"], arrs["gemm_C"] = A, B, om.gemm(A, B)
    arrs["gemm_kat"] = om.gemm(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0], [6.0]]))
    np.savez_compressed(os.path.join(OUT, "conv.npz"), **arrs)

    # 3. TinyCNN: data, init, one batch's loss and gradient (problems.py:152-275)
    arrs = {}
    for tag, (size, classes, n_ex, b) in {"s8c4": (8, 4, 64, 16), "s16c10": (16, 10, 128, 32)}.items():
        prob = om.make_tiny_cnn(size, classes, seed=3, n_examples=n_ex)
        W0 = prob.initial_weights()
        batch = prob.sample_batch(om.sgd.batch_stream(3), b)
        arrs[f"{tag}_meta"] = np.array([size, classes, n_ex, b, 3])
        arrs[f"{tag}_images"], arrs[f"{tag}_labels"] = prob.images, prob.labels
        arrs[f"{tag}_W0"] = W0
        arrs[f"{tag}_bx"], arrs[f"{tag}_by"] = batch
        arrs[f"{tag}_loss"] = np.array(prob.loss(W0, batch))
        arrs[f"{tag}_grad"] = prob.grad(W0, batch)
        arrs[f"{tag}_full_loss"] = np.array(prob.full_loss(W0))
    # 4. run_sync: 8 steps, sample every step (sgd.py:210-256)
    prob = om.make_tiny_cnn(8, 4, seed=3, n_examples=64)
    hp = om.Hyperparams(eta=0.05, mu=0.9, lam=1e-3, b=16)
    tr = om.run_sync(prob, hp, prob.initial_state(), om.StopRule(max_steps=8), seed=11)
    arrs["sync_hp"] = np.array([0.05, 0.9, 1e-3, 16, 8, 11])
    arrs["sync_W"], arrs["sync_V"], arrs["sync_losses"] = tr.final_state.W, tr.final_state.V, tr.losses
    # 5. simulate, deterministic, g = 4, 12 updates (simulator.py:123-213)
    plan = om.ExecutionPlan(N=8, g=4)
    prof = om.PhaseProfile(T_cc=8.0, T_nc=0.1, t_fc=0.5)
    cfg = om.SimConfig(plan=plan, profile=prof, hp=hp, problem=prob, max_updates=12, seed=5)
    st = om.simulate(cfg)
    arrs["sim_W"], arrs["sim_V"] = st.final_state.W, st.final_state.V
    arrs["sim_events"] = np.array([[e.group_id, e.read_step, e.write_step, e.staleness,
                                    e.start_time, e.fc_enqueue_time, e.finish_time] for e in st.events])
    arrs["sim_losses"] = st.loss_values
    cfg_e = om.SimConfig(plan=om.ExecutionPlan(N=8, g=8), profile=prof, hp=hp, problem=prob,
                         service_mode="exponential", max_updates=20, seed=7)
    st = om.simulate(cfg_e)
    arrs["simexp_events"] = np.array([[e.group_id, e.read_step, e.write_step, e.staleness,
                                       e.start_time, e.fc_enqueue_time, e.finish_time] for e in st.events])
    arrs["simexp_W"] = st.final_state.W
    # 6. sgd_step KATs
    s = om.sgd_step(om.SGDState(W=np.array([1.0]), V=np.array([0.0])), om.Hyperparams(eta=0.1, mu=0.9),
                    np.array([2.0]), np.array([1.0]))
    arrs["sgd_kat"] = np.array([s.W[0], s.V[0]])
    np.savez_compressed(os.path.join(OUT, "tinycnn.npz"), **arrs)

    # 7. implicit-momentum estimator (simulator.py:244-321) on the TinyCNN,
    #    exponential service, explicit momentum 0, g = 2 and 4
    from omnisim.simulator import estimate_implicit_momentum

    arrs = {}
    prob = om.make_tiny_cnn(8, 4, seed=3, n_examples=64)
    hp0 = om.Hyperparams(eta=0.05, mu=0.0, lam=0.0, b=8)
    prof0 = om.PhaseProfile(T_cc=4.0, T_nc=0.0, t_fc=0.01)
    arrs["im_cfg"] = np.array([8, 4, 64, 3, 0.05, 8, 4.0, 0.01, 80, 3, 8])  # size classes n_ex seed eta b T_cc t_fc max_updates sim_seed n_runs
    for g in (2, 4):
        cfg = om.SimConfig(plan=om.ExecutionPlan(N=4, g=g), profile=prof0, hp=hp0, problem=prob,
                           service_mode="exponential", max_updates=80, seed=3)
        arrs[f"im_g{g}"] = np.array(estimate_implicit_momentum(cfg, n_runs=8))
    np.savez_compressed(os.path.join(OUT, "implicit_momentum.npz"), **arrs)
    print("wrote fixtures to", OUT)


if __name__ == "__main__":
    main()
