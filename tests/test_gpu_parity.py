"""GPU parity: every CUDA stage and the whole path against the CPU oracle
(which is itself pinned to the reference, tests/test_oracle_golden.py).

Integer / byte / index work is compared bit-exactly; decoded floats are
compared bit-exactly against the oracle's decoder AND checked against the
point-wise error bound.  Run on a B200: pytest -m gpu."""

import numpy as np
import pytest

from conftest import CPC_CASES, GOLDEN_CASES, golden_inputs, load_golden, sha

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import gpu_hooks as H  # noqa: E402
import paper_1711_03888_b200 as nbz  # noqa: E402
from paper_1711_03888_b200 import datagen  # noqa: E402

REL4 = nbz.ErrorBoundSpec.relative(1e-4)


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


@pytest.fixture(params=["warp", "thread"])
def encoder(request, monkeypatch):
    """Both v2 payload encoders (warp-per-chunk with look-back,
    thread-per-chunk after a chunk-bit scan); csrc/encode.cu picks by chunk
    count unless NBZG_ENCODE forces one."""
    monkeypatch.setenv("NBZG_ENCODE", request.param)
    return request.param


@pytest.fixture(params=["warp", "thread"])
def decoder(request, monkeypatch):
    """Both v2 decoders (warp-per-chunk with resync, thread-per-chunk);
    csrc/decode.cu picks by chunk count unless NBZG_DECODE forces one."""
    monkeypatch.setenv("NBZG_DECODE", request.param)
    return request.param


# ---------------------------------------------------------------- stages

def test_minmax6(rng):
    fields = [rng.normal(0, 100, 100003).astype(np.float32) for _ in range(6)]
    fields[2][5] = -0.0
    mm = H.minmax6(fields)
    for f in range(6):
        assert mm[2 * f] == fields[f].min() and mm[2 * f + 1] == fields[f].max()


def test_integerize_matches_oracle(O, rng):
    for b in (0.0256, 0.05, 1e-3, 0.125, 7.0):
        x = rng.normal(0, 300, 200000).astype(np.float32)
        # exact half-integer ties and near-ties of x / 2b
        t = np.arange(-5000, 5000) + 0.5
        x[:10000] = (t * 2 * b).astype(np.float32)
        x[10000:20000] = np.nextafter(x[:10000], np.float32(np.inf))
        got, st = H.integerize(x, b)
        assert st == 0
        assert np.array_equal(got, O.integerize(x, b)), b
    got, st = H.integerize(np.array([1e30, 1.0], np.float32), 1e-12)
    assert st == nbz_status("bound too small")


def nbz_status(name):
    from paper_1711_03888_b200 import _native as N
    return {v: k for k, v in N.STATUS_NAMES.items()}[name]


@pytest.mark.parametrize("case", ["hacc34", "amdf40k", "sweep_hacc20", "sweep_amdf8k", "tiny3",
                                  "const2", "noise20k"])
def test_rindex_keys_and_order(O, case):
    g = load_golden(case)
    fields = golden_inputs(g)
    n = fields[0].size
    for tag in g["tags"]:
        t = str(tag)
        if not t.startswith("sz-lv-prx"):
            continue
        bounds = g[f"{t}|bounds"]
        mask = int(g[f"{t}|mask"])
        b3 = [0.0 if mask & (1 << i) else bounds[i] for i in range(3)]
        keys, bits, st = H.rindex_keys(fields[:3], b3)
        assert st == 0
        cols = [O.integerize(fields[i], bounds[i]) if not mask & (1 << i)
                else np.zeros(n, np.int64) for i in range(3)]
        okeys, obits, _ = O.build_rindex(cols, 16384)
        assert np.array_equal(keys, okeys), t
        assert np.array_equal(bits, obits), t
        if f"{t}|keys_sha" in g:
            assert sha(keys) == str(g[f"{t}|keys_sha"])
        order = H.prx_order(keys, 16384, bits, 6)
        assert np.array_equal(order, O.prx_order(okeys, 16384, obits, 6)), t
        for k in (0, 2, 4, 8):
            assert np.array_equal(H.prx_order(keys, 16384, bits, k),
                                  O.prx_order(okeys, 16384, obits, k)), (t, k)


def test_huffman_lengths_kats(O):
    k = load_golden("kats")
    for i in (1, 2, 3):
        got, st = H.huffman_lengths(k[f"hl_c{i}"])
        assert st == 0
        assert np.array_equal(got.astype(np.int64), k[f"hl_l{i}"]), i


def test_huffman_lengths_random(O, rng):
    for kk in (2, 3, 17, 300, 5000, 16384, 20000, 65536):
        c = np.sort(rng.integers(1, 10 ** 5, kk)).astype(np.int64)
        got, st = H.huffman_lengths(c)
        assert st == 0
        assert np.array_equal(got.astype(np.int64), O.huffman_lengths(c)), kk
    # heavy ties (leaf-wins-ties rule matters)
    c = np.sort(np.repeat(np.arange(1, 40), 97)).astype(np.int64)
    got, _ = H.huffman_lengths(c)
    assert np.array_equal(got.astype(np.int64), O.huffman_lengths(c))


def test_codebook_matches_oracle(O, rng):
    for nsym, spread in ((200, 30.0), (5000, 900.0), (30000, 9000.0)):
        codes = np.clip(np.rint(rng.normal(32769, spread, 400000)), 1, 65535).astype(np.int64)
        codes[::997] = 0
        hist = np.bincount(codes, minlength=65536)
        sym, lens, lut, m = H.huffman_codebook(hist)
        osym, olens = O.huffman_build(hist)
        assert np.array_equal(sym, osym)
        assert np.array_equal(lens, olens)
        tabs = O.huffman_tables(osym, olens)
        assert np.array_equal(lut[osym], tabs["enc_packed"][osym])
        assert m.f[0].total_bits == int((hist[osym] * olens.astype(np.int64)).sum()) + 32 * int(hist[0])
        assert m.f[0].n_esc == hist[0]


def test_huff_encode_bytes_match_reference_kat(O):
    k = load_golden("kats")
    syms = k["hb_syms_in"].astype(np.uint16)
    tabs = O.huffman_tables(k["hb_symbols"], k["hb_lengths"])
    lut = np.zeros(65536, np.uint64)
    lut[:tabs["enc_packed"].size] = tabs["enc_packed"]
    data, bits, _ = H.huff_encode(syms, lut)
    assert bits == int(k["hb_bits"])
    assert data == k["hb_bytes"].tobytes()


def test_huff_decode_hook_matches_reference_kat(O, rng):
    """K.huff_decode parity hook: the reference's KAT bitstream decodes to
    its symbols; truncated and invalid streams give the reference's
    statuses (2 / 1 -> NBZG_TRUNCATED / NBZG_INVALID_CODE)."""
    k = load_golden("kats")
    syms, lens = k["hb_symbols"], k["hb_lengths"]
    t = O.huffman_tables(syms, lens)
    data = k["hb_bytes"].tobytes()
    n = k["hb_syms_in"].size
    out, st = H.huff_decode(data, int(k["hb_bits"]), n, t)
    assert st == 0
    assert np.array_equal(out, k["hb_syms_in"])
    _o, st = H.huff_decode(data, int(k["hb_bits"]) - 3, n, t)
    assert st == 4  # NBZG_TRUNCATED
    # an incomplete code: one length-2 symbol only leaves "1..." invalid
    t2 = O.huffman_tables(np.array([5], np.int32), np.array([2], np.uint8))
    _o, st = H.huff_decode(b"\xff\xff", 16, 4, t2)
    assert st == 3  # NBZG_INVALID_CODE


def test_deinterleave3_hook(O):
    """K.deinterleave3 hook inverts the reference's interleave3 KAT."""
    k = load_golden("kats")
    x, y, z = H.deinterleave3(k["il_keys"])
    assert np.array_equal(x, k["il_x"]) and np.array_equal(y, k["il_y"])
    assert np.array_equal(z, k["il_z"])


def test_huff_encode_multichunk(O, rng):
    for n in (16383, 16384, 16385, 100000, 333333):
        codes = np.clip(np.rint(rng.normal(32769, 40, n)), 1, 65535).astype(np.int64)
        codes[::61] = rng.integers(1, 65535, codes[::61].size)
        hist = np.bincount(codes, minlength=65536)
        osym, olens = O.huffman_build(hist)
        tabs = O.huffman_tables(osym, olens)
        lut = np.zeros(65536, np.uint64)
        lut[:tabs["enc_packed"].size] = tabs["enc_packed"]
        data, bits, cb = H.huff_encode(codes.astype(np.uint16), lut)
        odata, obits = O.huff_encode(codes.astype(np.int32), tabs["enc_packed"])
        assert bits == obits and data == odata, n
        lens = (tabs["enc_packed"][codes] >> np.uint64(57)).astype(np.int64)
        want = [int(lens[i:i + 16384].sum()) for i in range(0, n, 16384)]
        assert list(cb) == want


def test_crc64(O, rng):
    assert H.crc64(b"123456789") == 0x995DC9BBDF1939FA
    for n in (0, 1, 7, 1023, 1024, 1025, 2047, 2048, 2049, 100003, 3 << 20, (512 << 10) * 3 + 5):
        b = rng.integers(0, 256, n).astype(np.uint8).tobytes()
        assert H.crc64(b) == O.crc64(b), n


def test_crc64_unaligned_and_batched(O, rng):
    """Device ranges at every 16-byte misalignment, several queued with one
    readback (crc64_device_many), and one range long enough (> 1024 spans of
    512 KiB) for the fold kernel's sequential runs."""
    import torch
    from paper_1711_03888_b200 import io as nio
    big = rng.integers(0, 256, (1 << 29) + (3 << 19) + 77).astype(np.uint8)
    d = torch.from_numpy(big).cuda()
    parts, want = [], []
    for off in range(16):
        ln = 70001 + 13 * off
        parts.append((d[off:off + ln], ln))
        want.append(O.crc64(big[off:off + ln].tobytes()))
    assert nio.crc64_device_many(parts) == want
    assert nio.crc64_device(d[5:], big.size - 5) == O.crc64(big[5:].tobytes())


# ---------------------------------------------------------------- whole path

@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_archive_byte_identical_to_oracle(O, case, encoder):
    """The GPU v2 archive equals the oracle's v2 archive byte for byte:
    bounds, seg bits, permutation, dual-quant codes, Huffman tables, chunk
    index, bitstream, escapes, CRCs, header."""
    g = load_golden(case)
    fields = golden_inputs(g)
    snap = nbz.ParticleSnapshot(*fields)
    for tag in g["tags"]:
        mode, eb = str(tag).split("|")
        res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(float(eb)))
        ref = O.compress(fields, mode, "rel", float(eb), fmt=2)
        assert tuple(res.archive.bounds) == tuple(ref["bounds"]), tag
        assert res.archive.constant_mask == ref["mask"]
        if mode == "sz-lv-prx" and snap.n:
            assert np.array_equal(res.archive.seg_bits, ref["seg_bits"]), tag
            assert np.array_equal(res.order, ref["order"]), tag
            if f"{tag}|order_sha" in g:
                assert sha(res.order.astype(np.int64)) == str(g[f"{tag}|order_sha"])
        for st in res.archive.streams:
            assert st.payload == ref["payloads"][st.field], (tag, st.field)
        wire = res.archive.serialized()
        assert wire == ref["wire"], tag
        assert res.archive.total_bytes() == len(wire)
        # ratio within 0.5% of the REFERENCE's (golden) ratio
        if snap.n >= 1000:
            r = nbz.ratio(res.archive)
            assert abs(r / float(g[f"{tag}|ratio"]) - 1) < 0.005, (tag, r)


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_decompress_matches_oracle_and_bound(O, case, decoder):
    g = load_golden(case)
    fields = golden_inputs(g)
    snap = nbz.ParticleSnapshot(*fields)
    for tag in g["tags"]:
        mode, eb = str(tag).split("|")
        res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(float(eb)))
        recon = nbz.decompress(res.archive)
        ref = O.compress(fields, mode, "rel", float(eb), fmt=2)
        odec = O.decompress(ref["wire"])
        work = fields if res.order is None else [f[res.order] for f in fields]
        for fi in range(6):
            got = np.asarray(recon.field(fi))
            assert np.array_equal(got, odec[fi]), (tag, fi)
            err = np.abs(work[fi].astype(np.float64) - got.astype(np.float64))
            lim = res.archive.bounds[fi] if not res.archive.is_constant(fi) else 0.0
            assert float(err.max(initial=0.0)) <= lim, (tag, fi)


@pytest.mark.parametrize("case", ["hacc34", "amdf40k", "sweep_hacc20", "const2", "noise20k"])
def test_reference_v1_archives_decode(O, case):
    """Archives written by the reference (v1, exact chain) decode on the GPU
    to exactly the reference's decompressed values (golden SHA-256)."""
    from paper_1711_03888_b200 import io as nio
    g = load_golden(case)
    fields = golden_inputs(g)
    for tag in g["tags"]:
        mode, eb = str(tag).split("|")
        wire = O.compress(fields, mode, "rel", float(eb), fmt=1)["wire"]
        assert sha(wire) == str(g[f"{tag}|wire_sha"])  # this IS the reference's archive
        ar = nio.deserialize_archive(wire)
        assert ar.version == 1
        recon = nbz.decompress(ar)
        for fi in range(6):
            key = f"{tag}|recon{fi}_sha"
            if key in g:
                assert sha(np.asarray(recon.field(fi))) == str(g[key]), (tag, fi)
        assert nio.serialize_archive(ar) == wire


def test_wire_round_trip_and_device_input(O):
    from paper_1711_03888_b200 import io as nio
    fields = datagen.small_amdf(70000)
    snap = nbz.ParticleSnapshot(*fields)
    res = nbz.compress(snap, "sz-lv-prx", REL4)
    wire = res.archive.serialized()
    again = nio.deserialize_archive(wire)
    assert nio.serialize_archive(again) == wire
    a = nbz.decompress(res.archive)
    b = nbz.decompress(again)
    for x, y in zip(a.fields(), b.fields()):
        assert np.array_equal(np.asarray(x), np.asarray(y))
    # in-situ: CUDA tensors in, CUDA tensors out, same bytes
    dsnap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
    dres = nbz.compress(dsnap, "sz-lv-prx", REL4)
    assert dres.archive.serialized() == wire
    drec = nbz.decompress(dres.archive)
    assert drec.on_device
    assert np.array_equal(drec.xx.cpu().numpy(), np.asarray(a.xx))


# ---------------------------------------------------------------- edge cases

def test_empty_snapshot():
    res = nbz.compress(nbz.ParticleSnapshot.empty(), "sz-lv-prx", REL4)
    assert res.archive.n == 0 and res.archive.streams == ()
    assert nbz.ratio(res.archive) is None
    out = nbz.decompress(res.archive)
    assert out.n == 0


@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 9, 100, 16383, 16385])
def test_tiny_and_ragged(O, rng, n):
    fields = [rng.uniform(0, 100, n).astype(np.float32) for _ in range(3)]
    fields += [rng.normal(0, 300, n).astype(np.float32) for _ in range(3)]
    snap = nbz.ParticleSnapshot(*fields)
    for mode in ("sz-lv", "sz-lv-prx"):
        res = nbz.compress(snap, mode, REL4)
        ref = O.compress(fields, mode, "rel", 1e-4, fmt=2)
        assert res.archive.serialized() == ref["wire"], (mode, n)
        rec = nbz.decompress(res.archive)
        odec = O.decompress(ref["wire"])
        for fi in range(6):
            assert np.array_equal(np.asarray(rec.field(fi)), odec[fi])


def test_constant_fields_and_absolute_bounds(O, rng):
    n = 40000
    fields = [rng.uniform(0, 100, n).astype(np.float32) for _ in range(6)]
    fields[0][:] = 3.25
    fields[5][:] = -1.0
    snap = nbz.ParticleSnapshot(*fields)
    bounds = {name: nbz.ErrorBoundSpec.absolute(0.01) for name in nbz.FIELD_NAMES}
    for mode in ("sz-lv", "sz-lv-prx"):
        res = nbz.compress(snap, mode, bounds)
        assert res.archive.constant_mask == 0b100001
        ref = O.compress(fields, mode, "abs", 0.01, fmt=2)
        assert res.archive.serialized() == ref["wire"]
        rec = nbz.decompress(res.archive)
        assert np.all(np.asarray(rec.xx) == np.float32(3.25))


def test_escape_heavy_and_tight_bounds(O, rng, decoder, encoder):
    n = 50000
    fields = [(rng.standard_cauchy(n) * 50).astype(np.float32) for _ in range(6)]
    snap = nbz.ParticleSnapshot(*fields)
    for eb in (1e-4, 1e-6, 1e-7):
        for mode in ("sz-lv", "sz-lv-prx"):
            res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(eb))
            ref = O.compress(fields, mode, "rel", eb, fmt=2)
            assert res.archive.serialized() == ref["wire"], (eb, mode)
            rec = nbz.decompress(res.archive)
            odec = O.decompress(ref["wire"])
            work = fields if res.order is None else [f[res.order] for f in fields]
            for fi in range(6):
                got = np.asarray(rec.field(fi))
                assert np.array_equal(got, odec[fi]), (eb, mode, fi)
                err = np.abs(work[fi].astype(np.float64) - got.astype(np.float64))
                assert float(err.max()) <= res.archive.bounds[fi]


def test_deferred_far_code_histogram(O, rng, monkeypatch):
    """Large alphabets: once a quantise CTA has spent its budget of global
    histogram atomics, the far codes of its remaining tiles are counted from
    the stored codes in shared memory (quant.cu).  A budget of 64 makes every
    CTA with more than one tile switch: archives still byte-identical."""
    monkeypatch.setenv("NBZG_Q_FAR_BUDGET", "64")
    n = 6_000_000  # 367 tiles per field over <= 49 CTAs: several tiles per CTA
    fields = [(rng.standard_normal(n) * (10.0 ** (f % 3))).astype(np.float32) for f in range(6)]
    snap = nbz.ParticleSnapshot(*fields)
    for mode in ("sz-lv", "sz-lv-prx"):
        res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(2e-6))
        ref = O.compress(fields, mode, "rel", 2e-6, fmt=2)
        assert res.archive.serialized() == ref["wire"], mode


def test_bound_too_small_raises():
    x = np.array([1e30, -1e30, 5.0, 7.0], np.float32)
    snap = nbz.ParticleSnapshot(x, x, x, x, x, x)
    with pytest.raises(nbz.BoundTooSmallError):
        nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.absolute(1e-30))


# ---------------------------------------------------------------- CPC2000 family

@pytest.mark.parametrize("case", CPC_CASES)
def test_cpc_archive_byte_identical_to_oracle(O, case):
    """sz-cpc2000 / cpc2000 on the GPU: full-key sort (k = 0, no clamp),
    segment minima, coordinate stream (raw first key + unsigned VLC deltas,
    per-segment scheme, corrections), SZ or signed-VLC velocities; the v2
    archive equals the oracle's byte for byte, and decoding it (and the
    REFERENCE's own v1 archive) gives the oracle's / reference's values."""
    g = load_golden(case)
    fields = golden_inputs(g)
    ss = int(g["segment_size"])
    settings = nbz.Settings(segment_size=ss)
    snap = nbz.ParticleSnapshot(*fields)
    for tag in g["tags"]:
        t = str(tag)
        mode, eb = t.split("|")
        res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(float(eb)), settings)
        ref = O.compress_cpc(fields, mode, "rel", float(eb), segment_size=ss, fmt=2)
        assert np.array_equal(res.order, ref["order"]), tag
        wire = res.archive.serialized()
        assert wire == ref["wire"], tag
        assert res.archive.total_bytes() == len(wire)
        out = nbz.decompress(res.archive)
        odec = O.decompress_cpc(ref["wire"])
        for fi in range(6):
            assert np.array_equal(np.asarray(out.field(fi)).view(np.uint32),
                                  odec[fi].view(np.uint32)), (tag, fi)
            if not res.archive.is_constant(fi):
                err = np.abs(fields[fi][ref["order"]].astype(np.float64)
                             - np.asarray(out.field(fi)).astype(np.float64))
                assert float(err.max()) <= res.archive.bounds[fi], (tag, fi)
        # the reference's own (v1) archive decodes on the GPU to its values
        from paper_1711_03888_b200 import io as nio
        ar1 = nio.deserialize_archive(bytes(g[f"{t}|wire"]))
        out1 = nbz.decompress(ar1)
        for fi in range(6):
            assert np.array_equal(np.asarray(out1.field(fi)).view(np.uint32),
                                  g[f"{t}|recon{fi}"].view(np.uint32)), (tag, fi, "v1")
        # v2 round trip through the wire
        out2 = nbz.decompress(nio.deserialize_archive(wire))
        for fi in range(6):
            assert np.array_equal(np.asarray(out2.field(fi)), np.asarray(out.field(fi))), (tag, fi)


@pytest.mark.parametrize("mode", ["sz-cpc2000", "cpc2000"])
def test_cpc_edge_cases(O, mode):
    """CPC modes: all three coordinates constant (no coordinate stream),
    a constant velocity, an empty snapshot, and a ragged multi-segment tile
    (segment 3000: 5 segments per tile) -- each byte-identical to the oracle
    and decoded exactly."""
    rng = np.random.default_rng(17)
    n = 20000
    f = [rng.uniform(0, 50, n).astype(np.float32) for _ in range(6)]
    cases = []
    g = list(f)
    g[0] = np.full(n, 1.5, np.float32)
    g[1] = np.full(n, -2.0, np.float32)
    g[2] = np.full(n, 3.25, np.float32)
    cases.append((g, 16384))
    h = list(f)
    h[4] = np.full(n, 9.0, np.float32)
    cases.append((h, 3000))
    cases.append(([np.zeros(0, np.float32)] * 6, 16384))
    for fields, ss in cases:
        snap = nbz.ParticleSnapshot(*fields)
        res = nbz.compress(snap, mode, REL4, nbz.Settings(segment_size=ss))
        ref = O.compress_cpc(fields, mode, "rel", 1e-4, segment_size=ss, fmt=2)
        wire = res.archive.serialized()
        assert wire == ref["wire"], (mode, ss)
        out = nbz.decompress(res.archive)
        if fields[0].size == 0:
            assert out.n == 0
            continue
        odec = O.decompress_cpc(ref["wire"])
        for fi in range(6):
            assert np.array_equal(np.asarray(out.field(fi)).view(np.uint32),
                                  odec[fi].view(np.uint32)), (mode, ss, fi)


def test_cpc_bound_too_small_raises():
    """No key clamp in the CPC modes: > 21 index bits per field raises
    BoundTooSmallError (rindex.py:185-190)."""
    rng = np.random.default_rng(3)
    f = [rng.uniform(0, 100, 5000).astype(np.float32) for _ in range(6)]
    snap = nbz.ParticleSnapshot(*f)
    for mode in ("cpc2000", "sz-cpc2000"):
        with pytest.raises(nbz.BoundTooSmallError):
            nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(1e-8))


def test_corrupt_archives_rejected():
    from paper_1711_03888_b200 import io as nio
    snap = nbz.ParticleSnapshot(*datagen.small_hacc(20))
    wire = nbz.compress(snap, "sz-lv-prx", REL4).archive.serialized()
    with pytest.raises(nbz.ArchiveError):
        nio.deserialize_archive(wire[:-1])
    with pytest.raises(nbz.ArchiveError):
        nio.deserialize_archive(b"XXXX" + wire[4:])
    rng = np.random.default_rng(5)
    for pos in rng.integers(0, len(wire), 40):
        bad = bytearray(wire)
        bad[pos] ^= 0x5A
        try:
            ar = nio.deserialize_archive(bytes(bad))
        except nbz.ArchiveError:
            continue
        nbz.decompress(ar)  # only reachable when the flip hit a CRC-neutral spot


def test_corrupt_payloads_fail_cleanly(decoder):
    """Bypass the CRC: hand-corrupted payloads must raise DecodeError (or
    decode to something), never hang or fault."""
    snap = nbz.ParticleSnapshot(*datagen.small_amdf(40000))
    res = nbz.compress(snap, "sz-lv", REL4)
    streams = res.archive.streams
    rng = np.random.default_rng(11)
    for trial in range(12):
        st = streams[trial % len(streams)]
        p = bytearray(st.payload)
        for pos in rng.integers(0, len(p), 3):
            p[pos] ^= int(rng.integers(1, 256))
        ar = nbz.Archive(res.archive.mode, res.archive.n, res.archive.interval_count,
                         res.archive.segment_size, res.archive.ignored_groups, None,
                         res.archive.bounds, res.archive.constant_mask, res.archive.constants,
                         streams=tuple(nbz.Stream(s.kind, s.field, bytes(p) if s is st else
                                                  s.payload) for s in streams))
        try:
            nbz.decompress(ar)
        except nbz.DecodeError:
            pass
    torch.cuda.synchronize()


# ---------------------------------------------------------------- larger sizes

@pytest.mark.parametrize("spec,mode", [("C1", "sz-lv"), ("C1", "sz-lv-prx"),
                                       ("C0", "sz-lv-prx")])
def test_config_scale_parity(O, spec, mode, decoder, encoder):
    """BASELINE configs 0 and 1 at full size: byte-identical archives."""
    fields = datagen.generate(spec)
    snap = nbz.ParticleSnapshot(*fields)
    res = nbz.compress(snap, mode, REL4)
    ref = O.compress(fields, mode, "rel", 1e-4, fmt=2)
    assert res.archive.serialized() == ref["wire"]
    rec = nbz.decompress(res.archive, device=True)
    odec = O.decompress(ref["wire"])
    work = fields if res.order is None else [f[res.order] for f in fields]
    for fi in range(6):
        got = rec.field(fi)
        assert torch.equal(got.cpu(), torch.from_numpy(odec[fi])), fi
        err = (torch.from_numpy(work[fi]).cuda().double() - got.double()).abs().max()
        assert float(err) <= res.archive.bounds[fi]


# ---------------------------------------------------------------- settings

@pytest.mark.parametrize("seg,ig,ic", [(1000, 6, 65536), (4099, 2, 65536), (16384, 0, 65536),
                                       (16384, 6, 1024), (777, 3, 4096), (16384, 6, 2)])
def test_settings_variants_byte_identical(O, seg, ig, ic, decoder, encoder):
    """Non-default Settings (segment size not a multiple of 4, ignored
    groups, small interval counts -> generic encoder path, heavy escapes):
    archives byte-identical to the oracle, decode exact and within bound."""
    fields = datagen.small_hacc(30)
    snap = nbz.ParticleSnapshot(*fields)
    settings = nbz.Settings(interval_count=ic, segment_size=seg, ignored_groups=ig)
    for mode in ("sz-lv", "sz-lv-prx"):
        res = nbz.compress(snap, mode, REL4, settings)
        ref = O.compress(fields, mode, "rel", 1e-4, interval_count=ic, segment_size=seg,
                         ignored_groups=ig, fmt=2)
        assert res.archive.serialized() == ref["wire"], (mode, seg, ig, ic)
        if res.order is not None:
            assert np.array_equal(res.order, ref["order"])
        rec = nbz.decompress(res.archive)
        odec = O.decompress(ref["wire"])
        work = fields if res.order is None else [f[res.order] for f in fields]
        for fi in range(6):
            got = np.asarray(rec.field(fi))
            assert np.array_equal(got, odec[fi]), (mode, fi)
            err = np.abs(work[fi].astype(np.float64) - got.astype(np.float64))
            assert float(err.max()) <= res.archive.bounds[fi]


@pytest.mark.parametrize("gen", ["hacc", "amdf", "C1"])
def test_auto_mode_keeps_smaller_archive(O, gen):
    """a13: snapshot-level auto policy = the smaller of sz-lv / sz-lv-prx,
    chosen from both modes' exact sizes before encoding (C1: the
    chunk-parallel encoder resumed after the sizing phase)."""
    fields = {"hacc": lambda: datagen.small_hacc(32), "amdf": lambda: datagen.small_amdf(40000),
              "C1": lambda: datagen.generate("C1")}[gen]()
    snap = nbz.ParticleSnapshot(*fields)
    a = nbz.compress(snap, "sz-lv", REL4).archive.serialized()
    b = nbz.compress(snap, "sz-lv-prx", REL4).archive.serialized()
    res = nbz.compress(snap, "auto", REL4)
    wire = res.archive.serialized()
    assert wire == (b if len(b) < len(a) else a)
    assert res.archive.mode.value in ("sz-lv", "sz-lv-prx")
    assert (res.order is not None) == (res.archive.mode.value == "sz-lv-prx")
    rec = nbz.decompress(res.archive)
    assert np.array_equal(np.asarray(rec.xx), O.decompress(wire)[0])


@pytest.mark.parametrize("eb", [1e-2, 1e-3, 1e-4, 1e-5, 1e-6])
@pytest.mark.parametrize("gen", ["hacc", "amdf"])
def test_config3_eb_sweep(O, eb, gen, decoder):
    """BASELINE config 3 shape (non-cubic HACC lattice / AMDF cells) at a
    reduced size, eb_rel 1e-2 ... 1e-6 (up to ~65K symbols, heavy escapes):
    byte-identical to the oracle, bound at every point, ratio within 0.5%
    of the reference algorithm's (oracle v1 = the reference's archive)."""
    if gen == "hacc":
        fields = datagen.generate(datagen.HaccSpec((128, 128, 64), 2.5, 7))
    else:
        fields = datagen.generate(datagen.AmdfSpec(1 << 20, seed=7))
    snap = nbz.ParticleSnapshot(*fields)
    for mode in ("sz-lv", "sz-lv-prx"):
        res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(eb))
        ref = O.compress(fields, mode, "rel", eb, fmt=2)
        wire = res.archive.serialized()
        assert wire == ref["wire"], (mode, eb)
        v1 = O.compress(fields, mode, "rel", eb, fmt=1)
        assert abs(nbz.ratio(res.archive) / v1["ratio"] - 1) < 0.005, (mode, eb)
        rec = nbz.decompress(res.archive, device=True)
        work = fields if res.order is None else [f[res.order] for f in fields]
        # (eb <= 1e-5: alphabets of 2^15-2^16 symbols -- the thread decoder's
        # canonical mode and the codebook's large-alphabet path)
        odec = O.decompress(ref["wire"])
        for fi in range(6):
            err = (torch.from_numpy(work[fi]).cuda().double() - rec.field(fi).double()).abs().max()
            lim = res.archive.bounds[fi] if not res.archive.is_constant(fi) else 0.0
            assert float(err) <= lim, (mode, eb, fi)
            assert np.array_equal(rec.field(fi).cpu().numpy(), odec[fi]), (mode, eb, fi)


@pytest.mark.parametrize("case", ["variants_hacc24", "variants_amdf20k"])
def test_rindex_variants_byte_identical(O, case):
    """Velocity and coord+velocity R-index variants (f4): GPU archives are
    byte-identical to the oracle's v2 archives (the oracle being pinned to
    the reference's keys / order / v1 archives for these variants)."""
    g = load_golden(case)
    fields = golden_inputs(g)
    S, ig = int(g["segment_size"]), int(g["ignored_groups"])
    snap = nbz.ParticleSnapshot(*fields)
    names = {"vel": nbz.RIndexVariant.VELOCITY, "coordvel": nbz.RIndexVariant.COORD_VELOCITY}
    for tag in g["tags"]:
        variant, eb = str(tag).split("|")
        settings = nbz.Settings(segment_size=S, ignored_groups=ig, rindex_variant=names[variant])
        res = nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.relative(float(eb)), settings)
        ref = O.compress(fields, "sz-lv-prx", "rel", float(eb), fmt=2, variant=variant,
                         segment_size=S, ignored_groups=ig)
        assert np.array_equal(res.order, ref["order"]), tag
        assert res.archive.serialized() == ref["wire"], tag
        rec = nbz.decompress(res.archive)
        odec = O.decompress(ref["wire"])
        for fi in range(6):
            assert np.array_equal(np.asarray(rec.field(fi)), odec[fi]), (tag, fi)
        # and the archive round-trips through the container
        from paper_1711_03888_b200 import io as nio
        assert nio.deserialize_archive(ref["wire"]).rindex_variant is names[variant]



@pytest.mark.parametrize("case", ["hacc34", "amdf40k", "noise20k", "lcf_hacc24", "lcf_noise20k"])
def test_sz_lcf_byte_identical_and_reference_v1_decode(O, case):
    """sz-lcf (LCF predictor, f4): GPU v2 archives byte-identical to the
    oracle's; the reference's own v1 sz-lcf archives (reproduced byte for
    byte by the pinned oracle) decode on the GPU to the reference's values."""
    g = load_golden(case)
    fields = golden_inputs(g)
    snap = nbz.ParticleSnapshot(*fields)
    for eb in (1e-4, 1e-6):
        res = nbz.compress(snap, "sz-lcf", nbz.ErrorBoundSpec.relative(eb))
        ref = O.compress(fields, "sz-lcf", "rel", eb, fmt=2)
        assert res.archive.serialized() == ref["wire"], (case, eb)
        rec = nbz.decompress(res.archive)
        odec = O.decompress(ref["wire"])
        for fi in range(6):
            got = np.asarray(rec.field(fi))
            assert np.array_equal(got, odec[fi]), (case, eb, fi)
            err = np.abs(fields[fi].astype(np.float64) - got.astype(np.float64))
            lim = res.archive.bounds[fi] if not res.archive.is_constant(fi) else 0.0
            assert float(err.max(initial=0.0)) <= lim
    if case.startswith("lcf_"):
        from paper_1711_03888_b200 import io as nio
        for tag in g["tags"]:
            t = str(tag)
            v1 = O.compress(fields, "sz-lcf", "rel", float(t.split("|")[1]), fmt=1)["wire"]
            assert sha(v1) == str(g[f"{t}|wire_sha"])
            out = nbz.decompress(nio.deserialize_archive(v1))
            for fi in range(6):
                assert sha(np.asarray(out.field(fi))) == str(g[f"{t}|recon{fi}_sha"]), (t, fi)


def test_sz_lcf_multichunk(O):
    """sz-lcf over many chunks (chain restart at every 16384 symbols)."""
    fields = datagen.generate("C1")
    snap = nbz.ParticleSnapshot(*fields)
    res = nbz.compress(snap, "sz-lcf", REL4)
    ref = O.compress(fields, "sz-lcf", "rel", 1e-4, fmt=2)
    assert res.archive.serialized() == ref["wire"]
    rec = nbz.decompress(res.archive, device=True)
    for fi in range(6):
        err = (torch.from_numpy(fields[fi]).cuda().double() - rec.field(fi).double()).abs().max()
        assert float(err) <= res.archive.bounds[fi]
