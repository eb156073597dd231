"""GPU parity of §8(f) f3: the 12-bit alphabet ("one 12-bit
channel, leading to 4096 possible shades of gray"; "our final model
has 4096 output layer neurons").  Readings R15-R17: features
v / 4096, P12 = 78 -> 256x5 -> 4096 (Table III ~1.35M), Q1' over 4096 symbols
with a 64-unit guard, u16 pixels, container byte 7 = 12.  Engine 3: P350K's
streamed layers plus a two-pass 4096-wide head (dlic_stream.cuh).

Bars as for the base network: logits within BF16_TOL of the
oracle's bf16 definition per row; integer tables equal to the oracle's Q1' of
the exported probabilities, which are the softmax of the exported logits to
fp32 accuracy; the production encoder's (f_s, c_s) equal to those tables;
containers byte-identical to the oracle coder fed the same (f_s, c_s);
lossless round trips."""

import numpy as np
import pytest

import synth
from oracle import codec, mlp, model_io, quant, window

pytestmark = pytest.mark.gpu

BF16_TOL = 8e-3
BF16_P90 = 1e-5


def _layers(seed=5):
    return synth.he_uniform_layers(mlp.P12, seed=seed, bias_scale=0.1)


def _img(h, w, seed):
    return synth.mri_like_volume(max(h, w), 1, seed=seed, bits=12)[0][:h, :w].copy()


@pytest.fixture(scope="module")
def dl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2207_05152_b200 as m
    return m


@pytest.fixture(scope="module")
def model(dl):
    blob = model_io.save(_layers())
    return blob, dl.dlic_model_load(blob, 0)


@pytest.mark.parametrize("h,w", [(13, 29), (40, 17)])
def test_12bit_logits_tables_vs_oracle(dl, model, h, w):
    blob, m = model
    img = _img(h, w, seed=h * w)
    img[0, 0], img[-1, -1] = 4095, 0
    out = dl.dlic_debug_mlp(m, img, precision=1)
    rows, cols = np.divmod(np.arange(h * w), w)
    ref = mlp.forward_bf16(_layers(), window.net_inputs(img, rows, cols, bits=12)).reshape(h, w, -1)
    lg = out["logits"]
    rel = np.abs(lg - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
    assert rel.max() <= BF16_TOL, float(rel.max())
    assert np.quantile(rel, 0.9) <= BF16_P90, float(np.quantile(rel, 0.9))
    # probabilities: the softmax of the GPU's own logits (fp32 accuracy)
    p_ref = quant.softmax_fp64(lg.reshape(-1, 4096))
    pg = out["probs"].reshape(-1, 4096)
    assert np.all(np.abs(pg - p_ref) <= 1e-5 * p_ref.max(-1, keepdims=True) + 1e-7)
    # integer tables: the oracle's Q1' (n = 4096, guard 64) of the GPU probabilities
    f = out["freqs"].astype(np.int64).reshape(-1, 4096)
    assert np.array_equal(f, quant.q1(pg))
    # the production encoder's (f_s, c_s) of the true symbols
    fc = dl.dlic_debug_mlp(m, img, precision=1, logits=False, probs=False, freqs=False)["fc"].reshape(-1)
    s = img.reshape(-1).astype(np.int64)
    c = quant.cdf(f)
    assert np.array_equal(fc & 0xFFFF, f[np.arange(len(s)), s]) and np.array_equal(fc >> 16, c[np.arange(len(s)), s])


@pytest.mark.parametrize("h,w,g,tile", [(20, 31, 32, (0, 0)), (33, 18, 4, (16, 10)), (1, 9, 32, (0, 0)),
                                        (70, 64, 8, (0, 0))])
def test_12bit_roundtrip_and_oracle_bytes(dl, model, h, w, g, tile):
    blob, m = model
    img = _img(h, w, seed=h + w)
    img[0, -1] = 4095
    bits = dl.dlic_encode(m, img, precision=1, group_rows=g, tile=tile)
    hd = dl.dlic_peek(bits)
    assert bits[7] == 12 and hd["bits"] == 12
    out = dl.dlic_decode(m, bits)
    assert out.dtype == np.uint16 and np.array_equal(out, img)
    fc = dl.dlic_debug_mlp(m, img, precision=1, group_rows=g, tile=tile, logits=False, probs=False,
                           freqs=False)["fc"]
    ob = codec.encode_with_tables((fc & 0xFFFF).astype(np.int64), (fc >> 16).astype(np.int64), w, h, 1, g,
                                  tile[0], tile[1], model_io.digest(blob), dl.dlic_numerics_rev(), bits=12)
    assert ob == bits


def test_12bit_edge_images(dl, model):
    _, m = model
    rng = np.random.default_rng(2)
    for img in (np.zeros((21, 40), np.uint16), np.full((5, 77), 4095, np.uint16),
                rng.integers(0, 4096, (66, 65), dtype=np.uint16)):
        assert np.array_equal(dl.dlic_decode(m, dl.dlic_encode(m, img)), img)


def test_12bit_batch_paths(dl, model):
    import torch
    _, m = model
    imgs = synth.mri_like_volume(96, 4, seed=9, bits=12)[:, :48, :80].copy()
    blobs, sizes = dl.dlic_encode_batch(m, imgs)
    off = 0
    for i in range(4):
        assert blobs[off:off + sizes[i]] == dl.dlic_encode(m, imgs[i])
        off += sizes[i]
    assert np.array_equal(dl.dlic_decode_batch(m, blobs, sizes), imgs)
    d_imgs = torch.from_numpy(imgs.view(np.int16)).cuda()      # u16 bytes in an int16 tensor
    d_out, d_sizes, stride = dl.dlic_encode_batch_device(m, d_imgs)
    torch.cuda.synchronize()
    sz = [int(x) for x in d_sizes.cpu()]
    hdr = dl.dlic_peek(d_out[:sz[0]].cpu().numpy().tobytes())
    d_dec = torch.empty_like(d_imgs)
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    dl.dlic_decode_batch_device(m, d_out, [i * stride for i in range(4)], sz, hdr, d_dec, st)
    torch.cuda.synchronize()
    assert st.cpu().tolist() == [0] * 4 and torch.equal(d_dec, d_imgs)


def test_12bit_rejections(dl, model):
    _, m = model
    img = _img(10, 12, seed=1)
    with pytest.raises(dl.DlicError) as e:
        dl.dlic_encode(m, img, precision=0)              # bf16 only
    assert e.value.status == 14
    m8 = dl.dlic_model_load(model_io.save(synth.he_uniform_layers(mlp.P350K, seed=3, bias_scale=0.1)), 0)
    b8 = dl.dlic_encode(m8, img.astype(np.uint8))
    with pytest.raises(dl.DlicError):                    # an 8-bit container with a 12-bit model
        dl.dlic_decode(m, b8)
