"""GPU parity of §8(f) f2: volumes with the 2-layer 3D window (P:204-205,
reading R13: the 78-tap window + the 3x3 box of the slice below) and the
overlapped 3D wavefront (R14): every slice's wavefront runs at
once, each slice's clusters waiting for the slice below through per-unit
progress flags.  The 9 lower taps enter layer 1 through the bias term
(add_w3d) in both the encoder and the decoder.  Bars as for 2D."""

import numpy as np
import pytest

import synth
from oracle import codec, container, model_io, mlp, quant, window

pytestmark = pytest.mark.gpu

BF16_TOL = 8e-3


@pytest.fixture(scope="module")
def dl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2207_05152_b200 as m
    return m


def _layers3d(seed=11, zero_lower=False):
    layers = synth.he_uniform_layers((87, 128, 128, 128, 128, 128, 256), seed=seed, bias_scale=0.1)
    if zero_lower:
        layers[0][0][78:87] = 0.0
    return layers


@pytest.fixture(scope="module")
def model3d(dl):
    blob = model_io.save(_layers3d())
    return blob, dl.dlic_model_load(blob, 0)


def _volume(d, h, w, seed=0):
    return synth.mri_like_volume(max(h, w), d, seed=seed)[:, :h, :w].copy()


def _oracle_logits(blob, vol, prec):
    layers = model_io.load(blob)
    d, h, w = vol.shape
    rows, cols = np.divmod(np.arange(h * w), w)
    out = []
    for z in range(d):
        x = window.net_inputs_3d(vol[z], None if z == 0 else vol[z - 1], rows, cols)
        out.append((mlp.forward_fp64 if prec == 0 else mlp.forward_bf16)(layers, x).reshape(h, w, 256))
    return np.stack(out)


@pytest.mark.parametrize("prec", [0, 1])
def test_volume_logits_vs_oracle(dl, model3d, prec):
    blob, m = model3d
    vol = _volume(3, 37, 61, seed=2)
    out = dl.dlic_debug_mlp(m, vol, precision=prec)
    ref = _oracle_logits(blob, vol, prec)
    rel = np.abs(out["logits"] - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
    assert rel.max() <= (1e-4 if prec == 0 else BF16_TOL), float(rel.max())
    assert np.array_equal(out["freqs"].astype(np.int64), quant.q1(out["probs"].reshape(-1, 256)).reshape(3, 37, 61, 256))


@pytest.mark.parametrize("prec", [1, 0])
@pytest.mark.parametrize("d,h,w,g,tile", [(1, 20, 30, 32, (0, 0)), (4, 40, 50, 8, (0, 0)), (3, 70, 45, 16, (24, 20)),
                                           (5, 9, 300, 32, (0, 0))])
def test_volume_roundtrip_and_oracle_bytes(dl, model3d, prec, d, h, w, g, tile):
    blob, m = model3d
    vol = _volume(d, h, w, seed=d + h)
    bits = dl.dlic_encode_volume(m, vol, precision=prec, group_rows=g, tile=tile)
    hd = dl.dlic_peek(bits)
    assert hd["depth"] == d and hd["n_streams"] % d == 0
    assert np.array_equal(dl.dlic_decode_volume(m, bits), vol)
    fc = dl.dlic_debug_mlp(m, vol, precision=prec, group_rows=g, tile=tile, logits=False, probs=False,
                           freqs=False)["fc"]
    ob = codec.encode_volume_with_tables((fc & 0xFFFF).astype(np.int64), (fc >> 16).astype(np.int64), w, h, prec, g,
                                         tile[0], tile[1], model_io.digest(blob), dl.dlic_numerics_rev())
    assert ob == bits
    assert container.parse(bits)["depth"] == d


def test_zero_lower_weights_match_the_2d_network_per_slice(dl):
    """With the lower layer's weights zero, add_w3d adds exact zeros: every
    slice's streams equal those of the 78-input network on that slice."""
    l3 = _layers3d(zero_lower=True)
    m3 = dl.dlic_model_load(model_io.save(l3), 0)
    l2 = [(l3[0][0][:78].copy(), l3[0][1])] + l3[1:]
    m2 = dl.dlic_model_load(model_io.save(l2), 0)
    vol = _volume(3, 33, 40, seed=5)
    hv = container.parse(dl.dlic_encode_volume(m3, vol))
    sps = container.streams_per_slice(40, 33, 0, 0, 32)
    for z in range(3):
        assert hv["streams"][z * sps:(z + 1) * sps] == container.parse(dl.dlic_encode(m2, vol[z]))["streams"]
    with pytest.raises(dl.DlicError) as e:      # a 3D model codes volumes only
        dl.dlic_encode(m3, vol[0])
    assert e.value.status == 2


def test_volume_tables_path_matches_oracle(dl):
    """rANS alone on volumes: GPU container == oracle's for the same tables;
    GPU table-fed decode of the oracle's container."""
    rng = np.random.default_rng(3)
    d, h, w = 3, 17, 23
    ft = np.zeros((d, h, w, 256), np.int64)
    vol = np.zeros((d, h, w), np.uint8)
    for idx in np.ndindex(d, h, w):
        p = rng.dirichlet(np.full(256, 0.3)).astype(np.float32)
        ft[idx] = quant.q1(p)
        vol[idx] = rng.choice(256, p=ft[idx] / 65536)
    ct = np.cumsum(ft, -1) - ft
    sym = vol.astype(np.int64)[..., None]
    fs = np.take_along_axis(ft, sym, -1)[..., 0]
    cs = np.take_along_axis(ct, sym, -1)[..., 0]
    sha = bytes(range(32))
    ob = codec.encode_volume_with_tables(fs, cs, w, h, 1, 8, 0, 0, sha, dl.dlic_numerics_rev())
    gb = dl.dlic_rans_encode_tables((fs | (cs << 16)).astype(np.uint32), precision=1, group_rows=8, model_sha=sha)
    assert gb == ob
    assert np.array_equal(dl.dlic_rans_decode_tables(ob, ft.astype(np.uint16)), vol)


def test_batch_of_volumes_device_api(dl, model3d):
    """Two volumes of 6 slices through the device batch API: one container per
    volume, all 12 slices' wavefronts in one launch (units ticketed in order)."""
    import torch
    blob, m = model3d
    vols = np.concatenate([_volume(6, 64, 80, seed=7), _volume(6, 64, 80, seed=8)])
    d_imgs = torch.from_numpy(vols).cuda()
    d_out, d_sizes, stride = dl.dlic_encode_batch_device(m, d_imgs, precision=1, volume_depth=6)
    torch.cuda.synchronize()
    sz = [int(x) for x in d_sizes.cpu()]
    assert len(sz) == 2
    host = d_out.cpu().numpy()
    for v in range(2):
        single = dl.dlic_encode_volume(m, vols[6 * v:6 * v + 6])
        assert host[v * stride:v * stride + sz[v]].tobytes() == single
    hdr = dl.dlic_peek(host[:sz[0]].tobytes())
    d_dec = torch.empty_like(d_imgs)
    st = torch.zeros(2, dtype=torch.int32, device="cuda")
    dl.dlic_decode_batch_device(m, d_out, [0, stride], sz, hdr, d_dec, st)
    torch.cuda.synchronize()
    assert st.cpu().tolist() == [0, 0] and torch.equal(d_dec, d_imgs)


def test_mri_volume_full_size(dl, model3d):
    """C3's slices as one 256x256x32 volume (the paper's MRI coder)."""
    blob, m = model3d
    vol = synth.mri_like_volume(256, 32, seed=3)
    bits = dl.dlic_encode_volume(m, vol)
    assert np.array_equal(dl.dlic_decode_volume(m, bits), vol)
    fc = dl.dlic_debug_mlp(m, vol, logits=False, probs=False, freqs=False)["fc"]
    ob = codec.encode_volume_with_tables((fc & 0xFFFF).astype(np.int64), (fc >> 16).astype(np.int64), 256, 256, 1,
                                         32, 0, 0, model_io.digest(blob), dl.dlic_numerics_rev())
    assert ob == bits
