"""GPU parity of §8(f) f4: optional pooling layers (reading R11 = SPEC
S:249: average over contiguous groups after the activation) and metadata
input features (reading R12 = SPEC S:252: min-max normalised,
appended after the pixel features, stored uncompressed in the container).

The engines fold pooling into the next layer's weights at model load and the
metadata into a per-image layer-1 bias (k_meta_bias), so the test model
exercises both: P100K-pool-meta = (78 + 3) -> 128 -> [avg 2] -> 128 -> 128 ->
[avg 2] -> 128 -> 128 -> 256 (92,800 + 384 parameters), random He-uniform
weights with biases.  Bars as for the base network."""

import numpy as np
import pytest

import synth
from oracle import codec, container, mlp, model_io, window

pytestmark = pytest.mark.gpu

BF16_TOL = 8e-3
POOL = [2, 0, 2, 0, 0, 0]
RANGE = [(0.0, 2.0), (0.0, 10.0), (0.5, 6.0)]     # spacing / slice spacing / thickness-like
META = [0.9, 3.0, 1.25]


def _layers(seed=7, zero_meta=False):
    layers = synth.he_uniform_pooled(81, [128, 128, 128, 128, 128, 256], POOL, seed=seed, bias_scale=0.1)
    if zero_meta:
        layers[0][0][78:] = 0.0
    return layers


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
    blob = model_io.save(_layers(), pool=POOL, meta_range=RANGE)
    return blob, dl.dlic_model_load(blob, 0)


def _oracle_logits(blob, img, prec, meta):
    net = model_io.load_net(blob)
    h, w = img.shape
    rows, cols = np.divmod(np.arange(h * w), w)
    x = window.net_inputs(img, rows, cols, window.meta_features(meta, net["meta_range"]))
    f = mlp.forward_fp64 if prec == 0 else mlp.forward_bf16
    return f(net["layers"], x, net["pool"]).reshape(h, w, -1)


@pytest.mark.parametrize("prec", [0, 1])
def test_pooled_meta_logits_vs_oracle(dl, model, prec):
    blob, m = model
    img = synth.natural_like(61, 37, seed=11)
    out = dl.dlic_debug_mlp(m, img, precision=prec, meta=META)
    ref = _oracle_logits(blob, img, prec, META)
    rel = np.abs(out["logits"] - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
    assert rel.max() <= (1e-4 if prec == 0 else BF16_TOL), float(rel.max())
    # tables follow exactly from the exported probabilities
    from oracle import quant
    assert np.array_equal(out["freqs"].astype(np.int64), quant.q1(out["probs"].reshape(-1, 256)).reshape(37, 61, 256))


@pytest.mark.parametrize("prec", [1, 0])
@pytest.mark.parametrize("h,w,g,tile", [(40, 50, 32, (0, 0)), (70, 45, 8, (24, 20)), (1, 13, 32, (0, 0))])
def test_pooled_meta_roundtrip_and_oracle_bytes(dl, model, prec, h, w, g, tile):
    blob, m = model
    img = synth.natural_like(w, h, seed=h + w)
    bits = dl.dlic_encode(m, img, precision=prec, group_rows=g, tile=tile, meta=META)
    hd = dl.dlic_peek(bits)
    assert hd["n_meta"] == 3 and np.array_equal(hd["meta"], np.array(META, np.float32))
    assert np.array_equal(dl.dlic_decode(m, bits), img)          # metadata re-read from the container
    fc = dl.dlic_debug_mlp(m, img, precision=prec, group_rows=g, tile=tile, logits=False, probs=False,
                           freqs=False, meta=META)["fc"]
    ob = codec.encode_with_tables((fc & 0xFFFF).astype(np.int64), (fc >> 16).astype(np.int64), w, h, prec, g,
                                  tile[0], tile[1], model_io.digest(blob), dl.dlic_numerics_rev(), meta=META)
    assert ob == bits
    assert container.parse(bits)["meta"].tolist() == pytest.approx(META)


def test_metadata_changes_tables_and_zero_meta_weights_match_plain_model(dl):
    img = synth.natural_like(64, 48, seed=5)
    blob = model_io.save(_layers(), pool=POOL, meta_range=RANGE)
    m = dl.dlic_model_load(blob, 0)
    a = dl.dlic_encode(m, img, meta=META)
    b = dl.dlic_encode(m, img, meta=[0.1, 9.0, 5.0])
    assert a != b and np.array_equal(dl.dlic_decode(m, b), img)
    # zero metadata weights: the per-image bias is exactly b1, so the payload
    # equals that of the same network without metadata inputs
    lz = _layers(zero_meta=True)
    mz = dl.dlic_model_load(model_io.save(lz, pool=POOL, meta_range=RANGE), 0)
    plain = [(lz[0][0][:78].copy(), lz[0][1])] + lz[1:]
    mp = dl.dlic_model_load(model_io.save(plain, pool=POOL), 0)
    pz = dl.dlic_peek(za := dl.dlic_encode(mz, img, meta=META))
    pp = dl.dlic_peek(zp := dl.dlic_encode(mp, img))
    assert za[pz["header_bytes"]:] == zp[pp["header_bytes"]:]
    with pytest.raises(dl.DlicError) as e:      # metadata count must match the model's
        dl.dlic_encode(m, img, meta=[1.0])
    assert e.value.status == 2
    with pytest.raises(dl.DlicError):
        dl.dlic_encode(m, img)


def test_batch_paths_with_per_image_metadata(dl, model):
    import torch
    blob, m = model
    imgs = synth.mri_like_slices(4, 256, seed0=2)[:, :60, :70].copy()
    meta = np.array([[0.9, 3.0, 1.25], [1.1, 4.0, 2.0], [0.5, 2.5, 1.0], [1.9, 9.0, 5.5]], np.float32)
    blobs, sizes = dl.dlic_encode_batch(m, imgs, meta=meta)
    off = 0
    for i in range(4):
        single = dl.dlic_encode(m, imgs[i], meta=meta[i])
        assert blobs[off:off + sizes[i]] == single
        off += sizes[i]
    assert np.array_equal(dl.dlic_decode_batch(m, blobs, sizes), imgs)
    d_imgs = torch.from_numpy(imgs).cuda()
    d_out, d_sizes, stride = dl.dlic_encode_batch_device(m, d_imgs, meta=meta)
    torch.cuda.synchronize()
    sz = [int(x) for x in d_sizes.cpu()]
    hdr = dl.dlic_peek(d_out[:sz[0]].cpu().numpy().tobytes())
    d_dec = torch.empty_like(d_imgs)
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    dl.dlic_decode_batch_device(m, d_out, [i * stride for i in range(4)], sz, hdr, d_dec, st)
    torch.cuda.synchronize()
    assert st.cpu().tolist() == [0] * 4 and torch.equal(d_dec, d_imgs)
