"""Full-size properties on the GPU: BASELINE config 2 (640^3 = 262,144,000
HACC-like particles, 6.29 GB), the size the bench runs at.  The oracle cannot
replay the whole snapshot here, so the checks are the size-independent ones
(SURVEY.md §8d acceptance): the error bound at every point, keys / seg bits /
order bit-exact against the oracle on 64 random segments (with the snapshot's
global bounds), the serialized archive decoding to the same values, and the
ratio in range."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1711_03888_b200 as nbz  # noqa: E402
from paper_1711_03888_b200 import io as nio  # noqa: E402

SIDE = 640
SEG = 16384


def _hacc_c2(seed: int = 7):
    """On-device HACC-like snapshot with config 2's shape: a 640^3 lattice of
    spacing 2.5 in a [0, 1600) box in lexicographic order, Gaussian
    displacement (sigma 0.5) wrapped periodically; velocities a smoothed
    Gaussian field (sigma ~300)."""
    n = SIDE ** 3
    g = torch.Generator(device="cuda").manual_seed(seed)
    idx = torch.arange(n, device="cuda", dtype=torch.int64)
    lat = (idx // (SIDE * SIDE), (idx // SIDE) % SIDE, idx % SIDE)
    del idx
    out = []
    for a in lat:
        x = 2.5 * a.to(torch.float64)
        x += 0.5 * torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
        out.append(torch.remainder(x, 1600.0).to(torch.float32))
    del lat
    k = torch.ones(1, 1, 9, device="cuda") / 3.0
    for _ in range(3):
        r = torch.randn(n, generator=g, device="cuda")
        v = torch.nn.functional.conv1d(r.view(1, 1, -1), k, padding=4).view(-1)
        out.append((300.0 * v).contiguous())
    return out


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


@pytest.fixture(scope="module")
def snap_c2():
    fields = _hacc_c2()
    torch.cuda.synchronize()
    return nbz.ParticleSnapshot(*fields)


def _bound_everywhere(snap, res, rec):
    order = res.order_device()
    for fi in range(6):
        x = snap.field(fi)[order] if order is not None else snap.field(fi)
        err = (x.double() - rec.field(fi).double()).abs().max().item()
        assert err <= res.archive.bounds[fi], (fi, err, res.archive.bounds[fi])


def test_c2_sz_lv_prx(O, snap_c2):
    snap = snap_c2
    res = nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.relative(1e-4))
    rec = nbz.decompress(res.archive, device=True)
    _bound_everywhere(snap, res, rec)
    r = nbz.ratio(res.archive)
    assert 3.0 < r < 8.0, r
    # keys / seg bits / order on 64 random segments vs the oracle, with the
    # snapshot's global bounds
    rng = np.random.default_rng(11)
    segs = np.sort(rng.choice(SIDE ** 3 // SEG, 64, replace=False))
    order = res.order_device()
    seg_bits = res.archive.seg_bits
    b3 = res.archive.bounds[:3]
    for s in segs:
        lo = int(s) * SEG
        xs = [snap.field(c)[lo:lo + SEG].cpu().numpy() for c in range(3)]
        ints = [O.integerize(xs[c], b3[c]) for c in range(3)]
        keys, bits, _mn = O.build_rindex(ints, SEG)
        assert int(bits[0]) == int(seg_bits[s]), s
        o_ref = O.prx_order(keys, SEG, bits, 6)
        got = order[lo:lo + SEG].cpu().numpy() - lo
        assert np.array_equal(got, o_ref), s
    # the serialized archive (CRC-64, container) decodes to the same values
    wire = res.archive.serialized()
    assert len(wire) == res.archive.total_bytes()
    rec2 = nbz.decompress(nio.deserialize_archive(wire), device=True)
    for fi in range(6):
        assert torch.equal(rec2.field(fi), rec.field(fi)), fi


@pytest.mark.parametrize("mode", ["sz-cpc2000", "cpc2000"])
def test_c2_cpc_modes(snap_c2, mode):
    snap = snap_c2
    res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(1e-4))
    rec = nbz.decompress(res.archive, device=True)
    _bound_everywhere(snap, res, rec)
    rec2 = nbz.decompress(nio.deserialize_archive(res.archive.serialized()), device=True)
    for fi in range(6):
        assert torch.equal(rec2.field(fi), rec.field(fi)), (mode, fi)


@pytest.mark.parametrize("cfg", ["C0", "C1"])
def test_baseline_configs_byte_identical(O, cfg):
    """BASELINE configs 0 (HACC-like 100^3, the reference's CPU-runnable case)
    and 1 (AMDF-like 2^22), at their full sizes: every mode's GPU archive is
    byte-identical to the oracle's v2 archive and decodes to its values; the
    ratio is within 0.5% of the reference algorithm's (oracle v1)."""
    from paper_1711_03888_b200 import datagen
    fields = datagen.generate(cfg)
    snap = nbz.ParticleSnapshot(*fields)
    for mode in ("sz-lv", "sz-lv-prx", "sz-cpc2000", "cpc2000"):
        res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(1e-4))
        wire = res.archive.serialized()
        cpc = mode in ("sz-cpc2000", "cpc2000")
        ref = (O.compress_cpc if cpc else O.compress)(fields, mode, "rel", 1e-4, fmt=2)
        assert wire == ref["wire"], (cfg, mode)
        v1 = (O.compress_cpc if cpc else O.compress)(fields, mode, "rel", 1e-4, fmt=1)
        assert abs(nbz.ratio(res.archive) / v1["ratio"] - 1) < 0.005, (cfg, mode)
        out = nbz.decompress(res.archive)
        odec = (O.decompress_cpc if cpc else O.decompress)(ref["wire"])
        for fi in range(6):
            assert np.array_equal(np.asarray(out.field(fi)).view(np.uint32),
                                  odec[fi].view(np.uint32)), (cfg, mode, fi)


@pytest.mark.parametrize("const_fields", [(0, 1, 2), (3, 4, 5), (1, 4)])
def test_field_groups_with_constant_fields(O, const_fields):
    """Archives large enough for the two-field-group compress (>= 256
    chunks per field) with whole groups or single fields constant:
    byte-identical to the oracle, decoded exactly."""
    rng = np.random.default_rng(5)
    n = (1 << 22) + 1000
    fields = [rng.uniform(0, 100, n).astype(np.float32) for _ in range(6)]
    for f in const_fields:
        fields[f] = np.full(n, 2.5 + f, np.float32)
    snap = nbz.ParticleSnapshot(*fields)
    for mode in ("sz-lv", "sz-lv-prx"):
        res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(1e-4))
        ref = O.compress(fields, mode, "rel", 1e-4, fmt=2)
        assert res.archive.serialized() == ref["wire"], (mode, const_fields)
        out = nbz.decompress(res.archive)
        odec = O.decompress(ref["wire"])
        for fi in range(6):
            assert np.array_equal(np.asarray(out.field(fi)), odec[fi]), (mode, fi)
