"""Pins for oracle.quant (softmax, Q1) and oracle.mlp."""

import math

import numpy as np
import torch

from conftest import golden
from oracle import mlp, quant
import synth


def test_softmax_closed_forms():
    for ex in golden("spec_quant_softmax.json")["softmax"]:
        lg = np.array([math.log(2) if v == "ln2" else v for v in ex["logits"]], dtype=np.float64)
        assert np.allclose(quant.softmax_fp64(lg), ex["p"], rtol=0, atol=1e-15)
    # shift invariance and batch consistency
    rng = np.random.default_rng(0)
    z = rng.normal(size=(5, 256)) * 10
    assert np.allclose(quant.softmax_fp64(z), quant.softmax_fp64(z + 1000.0), atol=1e-14)
    assert np.array_equal(quant.softmax_fp64(np.stack([z[0], z[0]]))[1], quant.softmax_fp64(z[:1])[0])


def test_q1_hand_derived_examples():
    for ex in golden("spec_quant_softmax.json")["quantize_pdf"]:
        if ex["p"] == "uniform256":
            f = quant.q1(np.full(256, 1 / 256, np.float32), ex["k"])
            assert np.all(f[:255] == 255) and f[255] == 511
        else:
            assert list(quant.q1(np.array(ex["p"], np.float32), ex["k"])) == ex["f"]


def test_q1_invariants_and_loss():
    rng = np.random.default_rng(1)
    lim = golden("spec_quant_softmax.json")["max_added_cross_entropy_bits"]
    worst, rmin, rmax = 0.0, 1 << 20, -(1 << 20)
    for _ in range(2000):
        logits = rng.normal(size=256) * rng.choice([0.5, 2.0, 8.0])
        p = quant.softmax_fp64(logits).astype(np.float32)
        f = quant.q1(p)
        assert f.sum() == 65536 and f.min() >= 1
        # monotone in p below the residual slot: p_i > p_j => f_i >= f_j
        o = np.argsort(p[:255], kind="stable")
        assert np.all(np.diff(f[:255][o]) >= 0)
        base = 1 + np.floor(p * np.float32(65279)).astype(np.int64)
        r = 65536 - base.sum()
        assert f[255] == base[255] + r and np.array_equal(f[:255], base[:255])
        rmin, rmax = min(rmin, r), max(rmax, r)
        pd = p.astype(np.float64) / p.astype(np.float64).sum()
        ce_f = -(pd * np.log2(f / 65536)).sum()
        ce_p = -(pd * np.log2(np.maximum(pd, 1e-300))).sum()
        worst = max(worst, ce_f - ce_p)
    assert worst < lim
    assert 0 <= rmin and rmax <= 257


def test_q1_residual_never_negative_at_fp32_limits():
    # adversarial fp32 softmaxes whose sum exceeds 1 by rounding
    rng = np.random.default_rng(2)
    for _ in range(3000):
        p = rng.dirichlet(np.full(256, rng.choice([0.01, 1.0, 100.0]))).astype(np.float32)
        p = (p * np.float32(1 + 2 ** -22)).astype(np.float32)     # push the sum above 1
        assert float(p.astype(np.float64).sum()) <= 1 + 258 * 2 ** -24
        f = quant.q1(p)
        assert f.min() >= 1 and f.sum() == 65536


def test_cdf_is_exclusive_prefix_sum():
    f = np.array([3, 1, 4, 1, 5, 2])
    assert list(quant.cdf(f)) == [0, 3, 4, 8, 9, 14]


def test_param_counts_match_table_I():
    facts = golden("paper_facts.json")["params"]
    assert len(mlp.P100K) - 1 == facts["layers"] and mlp.P100K[-1] == facts["outputs"]
    assert mlp.n_params(mlp.P100K) == 109184
    assert mlp.n_params(mlp.P350K) == 349184
    assert abs(mlp.n_params(mlp.P100K) - facts["p100k_approx"]) / facts["p100k_approx"] < 0.1
    assert abs(mlp.n_params(mlp.P350K) - facts["p350k_approx"]) / facts["p350k_approx"] < 0.01
    assert mlp.flops_per_pixel(mlp.P100K) == 216576


def test_forward_hand_computed():
    # x=[1,2]; h = relu([1*1+2*2, 1*(-1)+2*0+1]) = [5, 0]; out = 5*1 + 0*(-3) + 0.5 = 5.5
    layers = [(np.array([[1, -1], [2, 0]], np.float32), np.array([0, 1], np.float32)),
              (np.array([[1], [-3]], np.float32), np.array([0.5], np.float32))]
    assert mlp.forward_fp64(layers, np.array([[1.0, 2.0]]))[0, 0] == 5.5
    # a negative pre-activation is clipped: x=[-1, 0] -> h=relu([-1, 2]) = [0, 2] -> -6 + .5
    assert mlp.forward_fp64(layers, np.array([[-1.0, 0.0]]))[0, 0] == -5.5
    assert mlp.forward_bf16(layers, np.array([[1.0, 2.0]]))[0, 0] == 5.5


def test_fp32_within_1e6_of_fp64():
    layers = synth.he_uniform_layers(mlp.P100K, seed=3, bias_scale=0.1)
    rng = np.random.default_rng(3)
    x = rng.integers(0, 256, size=(512, 78)) / 256.0
    a = mlp.forward_fp64(layers, x)
    b = mlp.forward_fp32(layers, x).astype(np.float64)
    rel = np.abs(a - b).max(axis=1) / np.maximum(np.abs(a).max(axis=1), 1e-6)
    assert rel.max() < 1e-6


def test_bf16_round_matches_torch():
    rng = np.random.default_rng(4)
    v = np.concatenate([rng.normal(size=20000) * 10.0 ** rng.integers(-6, 6, 20000),
                        1 + np.arange(-40, 40) * 2.0 ** -9])          # includes exact ties
    ref = torch.from_numpy(v.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(mlp.bf16_round(v), ref)


def test_bf16_path_equals_exact_when_everything_is_representable():
    # small-integer weights and v/256 inputs: every operand and activation is
    # exactly representable in bf16 -> the bf16 path must equal the fp64 forward.
    # (sparse inputs keep every partial sum a short dyadic: |k| <= 192 units of 2^-12)
    rng = np.random.default_rng(5)
    dims = (78, 8, 8, 4)
    layers = [(rng.integers(-1, 2, size=(dims[i], dims[i + 1])).astype(np.float32) / 4,
               rng.integers(-4, 5, size=dims[i + 1]).astype(np.float32) / 1024) for i in range(3)]
    x = np.zeros((64, 78))
    for row in x:
        row[rng.choice(78, 3, replace=False)] = rng.integers(0, 5, 3) / 256.0
    assert np.array_equal(mlp.forward_bf16(layers, x), mlp.forward_fp64(layers, x))
    # ... and a non-representable weight changes it (the rounding is really applied)
    layers[0][0][0, 0] = np.float32(1 + 2.0 ** -10)
    x[:, 0] = 1.0
    assert not np.array_equal(mlp.forward_bf16(layers, x), mlp.forward_fp64(layers, x))


def test_batch_consistency():
    layers = synth.he_uniform_layers(mlp.P100K, seed=6)
    rng = np.random.default_rng(6)
    x = rng.integers(0, 256, size=(300, 78)) / 256.0
    full = mlp.logits_path(layers, x, 0)
    for i in (0, 17, 299):
        assert np.array_equal(full[i], mlp.logits_path(layers, x[i:i + 1], 0)[0])


def test_bf16_hidden_activations_are_rerounded_hand_derived():
    # One hidden unit: z1 = 1*1 + 2^-9 = 1 + 2^-9 exactly (fp32).  bf16 has an
    # 8-bit significand, so the next representable value above 1 is 1 + 2^-7;
    # 1 + 2^-9 lies below the midpoint 1 + 2^-8 and rounds DOWN to 1.  The
    # output layer (weight 1, bias 0) therefore returns exactly 1.0.  Without
    # the re-rounding it would return 1 + 2^-9.
    layers = [(np.array([[1.0]], np.float32), np.array([2.0 ** -9], np.float32)),
              (np.array([[1.0]], np.float32), np.array([0.0], np.float32))]
    assert mlp.forward_bf16(layers, np.array([[1.0]]))[0, 0] == 1.0
    assert mlp.forward_fp64(layers, np.array([[1.0]]))[0, 0] == 1.0 + 2.0 ** -9
    # 1 + 3*2^-9 lies above the midpoint 1 + 2^-8 -> rounds UP to 1 + 2^-7
    layers[0] = (layers[0][0], np.array([3 * 2.0 ** -9], np.float32))
    assert mlp.forward_bf16(layers, np.array([[1.0]]))[0, 0] == 1.0 + 2.0 ** -7
    # the exact midpoint 1 + 2^-8 ties to even (1.0, significand ...0)
    layers[0] = (layers[0][0], np.array([2.0 ** -8], np.float32))
    assert mlp.forward_bf16(layers, np.array([[1.0]]))[0, 0] == 1.0


def test_bf16_bias_is_added_in_fp32_to_the_fp32_rounded_sum_hand_derived():
    # Output layer only: inputs (1, 2^-30) with weights (1, 1) are bf16-exact and
    # their exact sum is 1 + 2^-30, which rounds to 1.0 in fp32 (ulp 2^-23).
    # Adding the bias 2^-24 in fp32: 1 + 2^-24 is the midpoint of [1, 1 + 2^-23]
    # and ties to even -> exactly 1.0.  An fp64 bias add would give
    # 1 + 2^-24 + 2^-30, which is above the midpoint and rounds to 1 + 2^-23
    # when the logit is stored as fp32 (logits_path).
    layers = [(np.array([[1.0], [1.0]], np.float32), np.array([2.0 ** -24], np.float32))]
    x = np.array([[1.0, 2.0 ** -30]])
    assert mlp.forward_bf16(layers, x)[0, 0] == 1.0
    assert mlp.logits_path(layers, x, 1)[0, 0] == np.float32(1.0)
    assert mlp.logits_path(layers, x, 0)[0, 0] == np.float32(1.0 + 2.0 ** -23)    # fp64 path, for contrast
