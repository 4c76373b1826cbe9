"""Pin the CPU oracle to the reference: every golden vector in tests/golden/
was dumped from the reference package itself (scripts/make_golden.py).
CPU-only; no GPU needed."""

import numpy as np
import pytest

from conftest import CPC_CASES, GOLDEN_CASES, golden_inputs, load_golden, sha

MODES = {"sz-lv": "sz-lv", "sz-lv-prx": "sz-lv-prx"}


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_oracle_v1_archive_byte_identical(oracle_lib, case):
    O = oracle_lib
    g = load_golden(case)
    fields = golden_inputs(g)
    for tag in g["tags"]:
        mode, eb = str(tag).split("|")
        res = O.compress(fields, mode, "rel", float(eb), fmt=1)
        t = str(tag)
        assert np.array_equal(res["bounds"], g[f"{t}|bounds"]), tag
        assert res["mask"] == int(g[f"{t}|mask"]), tag
        if mode == "sz-lv-prx":
            assert np.array_equal(res["seg_bits"], g[f"{t}|seg_bits"]), tag
            if f"{t}|order_sha" in g:
                assert sha(res["order"].astype(np.int64)) == str(g[f"{t}|order_sha"]), tag
        for fi in range(6):
            key = f"{t}|payload{fi}_sha"
            if key in g:
                assert sha(res["payloads"][fi]) == str(g[key]), (tag, fi)
        assert sha(res["wire"]) == str(g[f"{t}|wire_sha"]), tag
        assert len(res["wire"]) == int(g[f"{t}|wire_len"])
        if res["ratio"] is not None:
            assert res["ratio"] == pytest.approx(float(g[f"{t}|ratio"]), rel=0, abs=0)


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_oracle_stages_match_reference(oracle_lib, case):
    """Keys, codes (exact chain), Huffman tables and the decoder output."""
    O = oracle_lib
    g = load_golden(case)
    fields = golden_inputs(g)
    n = fields[0].size
    for tag in g["tags"]:
        t = str(tag)
        mode, eb = t.split("|")
        bounds = g[f"{t}|bounds"]
        mask = int(g[f"{t}|mask"])
        if f"{t}|keys_sha" in g:
            cols = [O.integerize(fields[i], bounds[i]) if not mask & (1 << i)
                    else np.zeros(n, np.int64) for i in range(3)]
            keys, bits, _ = O.build_rindex(cols, 16384)
            assert sha(keys) == str(g[f"{t}|keys_sha"]), tag
            assert np.array_equal(bits, g[f"{t}|seg_bits"])
            order = O.prx_order(keys, 16384, bits, 6)
            work = [f[order] for f in fields]
        else:
            work = fields
        wire = O.compress(fields, mode, "rel", float(eb), fmt=1)["wire"]
        dec = O.decompress(wire)
        for fi in range(6):
            if f"{t}|codes{fi}_sha" not in g:
                continue
            codes, esc, _ = O.sz_quantize(work[fi], bounds[fi], 32768)
            assert sha(codes) == str(g[f"{t}|codes{fi}_sha"]), (tag, fi)
            assert esc.size == int(g[f"{t}|nesc{fi}"])
            syms, lens = O.huffman_build(np.bincount(codes))
            assert np.array_equal(syms, g[f"{t}|syms{fi}"]), (tag, fi)
            assert np.array_equal(lens, g[f"{t}|lens{fi}"]), (tag, fi)
        for fi in range(6):
            key = f"{t}|recon{fi}_sha"
            if key in g:
                assert sha(dec[fi]) == str(g[key]), (tag, fi)


def test_oracle_kats(oracle_lib):
    O = oracle_lib
    k = load_golden("kats")
    assert np.array_equal(O.interleave3(k["il_x"], k["il_y"], k["il_z"]), k["il_keys"])
    # field order KATs: xx is the most significant bit of each 3-bit group
    assert int(O.interleave3([1], [0], [0])[0]) == 0b100
    assert int(O.interleave3([0b11], [0], [0b11])[0]) == 0b101101
    assert np.array_equal(O.integerize(k["int_x"], float(k["int_b"])), k["int_out"])
    assert np.array_equal(O.integerize(k["int_x2"], 0.125), k["int_out2"])
    codes, esc, recon = O.sz_quantize(k["szq_x"], 0.01, 32768)
    assert np.array_equal(codes, k["szq_codes"])
    assert np.array_equal(recon, k["szq_recon"])
    assert np.array_equal(esc, k["szq_esc"])
    codes, esc, _ = O.sz_quantize(k["szq_x"], 0.01, 32768, use_lcf=True)
    assert np.array_equal(codes, k["szq_lcf_codes"])
    assert np.array_equal(esc, k["szq_lcf_esc"])
    back = O.sz_dequantize(k["szq_codes"], k["szq_esc"], 0.01, 32768)
    assert np.array_equal(back, k["szq_recon"])
    for i in (1, 2, 3):
        assert np.array_equal(O.huffman_lengths(k[f"hl_c{i}"]), k[f"hl_l{i}"]), i
    syms, lens = O.huffman_build(np.bincount(k["hb_syms_in"]))
    assert np.array_equal(syms, k["hb_symbols"])
    assert np.array_equal(lens, k["hb_lengths"])
    tabs = O.huffman_tables(syms, lens)
    data, bits = O.huff_encode(k["hb_syms_in"], tabs["enc_packed"])
    assert bits == int(k["hb_bits"])
    assert data == k["hb_bytes"].tobytes()
    back = O.huff_decode(data, bits, k["hb_syms_in"].size, tabs)
    assert np.array_equal(back, k["hb_syms_in"])
    assert O.crc64(b"123456789") == int(k["crc_123456789"]) == 0x995DC9BBDF1939FA
    assert O.crc64(k["crc_buf"].tobytes()) == int(k["crc_buf_val"])


def test_dual_quant_bound_and_roundtrip(oracle_lib, rng):
    """v2 dual-quant: error bound holds by construction; decode is exact."""
    O = oracle_lib
    for scale, b in [(100.0, 0.01), (300.0, 0.5), (1.0, 1e-6), (1e6, 1e-3)]:
        x = (np.cumsum(rng.normal(0, 1, 20000)) * scale / 100).astype(np.float32)
        x[::513] *= 1e4
        codes, esc, k_last = O.dq_quantize(x, b, 32768)
        y = O.dq_dequantize(codes, esc, b, 32768)
        assert np.all(np.abs(x.astype(np.float64) - y.astype(np.float64)) <= b)
        assert (codes == 0).sum() == esc.size
        # chaining over a split point with the carried k gives identical codes
        c0, _, _ = O.dq_quantize(x, b, 32768, chunk=0)
        c1, e1, k1 = O.dq_quantize(x[:7000], b, 32768, chunk=0)
        c2, e2, _ = O.dq_quantize(x[7000:], b, 32768, k_prev=k1, chunk=0)
        assert np.array_equal(np.concatenate([c1, c2]), c0)
        # with chunk restarts, each 16384-symbol chunk is independent
        for lo in range(0, x.size, 16384):
            cc, _, _ = O.dq_quantize(x[lo:lo + 16384], b, 32768, chunk=0)
            assert np.array_equal(cc, codes[lo:lo + 16384])


@pytest.mark.parametrize("case", ["hacc34", "amdf40k", "sweep_hacc20", "noise20k"])
def test_dual_quant_ratio_within_tolerance(oracle_lib, case):
    """v2 archives (dual-quant + chunk index) stay within 0.5% of the
    reference's compression ratio and decode within the bound."""
    O = oracle_lib
    g = load_golden(case)
    fields = golden_inputs(g)
    for tag in g["tags"]:
        t = str(tag)
        mode, eb = t.split("|")
        r2 = O.compress(fields, mode, "rel", float(eb), fmt=2)
        ref_ratio = float(g[f"{t}|ratio"])
        assert abs(r2["ratio"] / ref_ratio - 1.0) < 0.005, (tag, r2["ratio"], ref_ratio)
        dec = O.decompress(r2["wire"])
        work = fields if r2["order"] is None else [f[r2["order"]] for f in fields]
        for fi in range(6):
            err = np.abs(work[fi].astype(np.float64) - dec[fi].astype(np.float64))
            assert float(err.max()) <= r2["bounds"][fi] or r2["mask"] & (1 << fi)


@pytest.mark.parametrize("case", ["variants_hacc24", "variants_amdf20k"])
def test_oracle_rindex_variants_match_reference(oracle_lib, case):
    """Velocity and six-field coord+velocity R-index variants (rindex.py:24-44,
    interleave_any _kernels.py:801-810): keys, seg bits, order and the whole
    v1 archive byte-identical to the reference's."""
    O = oracle_lib
    g = load_golden(case)
    fields = golden_inputs(g)
    S, ig = int(g["segment_size"]), int(g["ignored_groups"])
    fi_of = {"vel": (3, 4, 5), "coordvel": (0, 1, 2, 3, 4, 5)}
    for tag in g["tags"]:
        t = str(tag)
        variant, eb = t.split("|")
        res = O.compress(fields, "sz-lv-prx", "rel", float(eb), fmt=1, variant=variant,
                         segment_size=S, ignored_groups=ig)
        assert np.array_equal(res["seg_bits"], g[f"{t}|seg_bits"]), t
        assert sha(res["order"].astype(np.int64)) == str(g[f"{t}|order_sha"]), t
        assert sha(res["wire"]) == str(g[f"{t}|wire_sha"]), t
        b, mask = g[f"{t}|bounds"], int(g[f"{t}|mask"])
        cols = [O.integerize(fields[i], b[i]) if not mask & (1 << i)
                else np.zeros(fields[0].size, np.int64) for i in fi_of[variant]]
        keys, bits, _ = O.build_rindex_n(cols, S)
        assert sha(keys) == str(g[f"{t}|keys_sha"]), t
        dec = O.decompress(res["wire"])
        for fi in range(6):
            assert sha(dec[fi]) == str(g[f"{t}|recon{fi}_sha"]), (t, fi)


@pytest.mark.parametrize("case", ["lcf_hacc24", "lcf_noise20k"])
def test_oracle_lcf_matches_reference(oracle_lib, case):
    """sz-lcf (LCF predictor pred = 2*prev - prev2, _kernels.py:162-165):
    v1 archives and decoded values byte-identical to the reference; the v2
    dual-quant restatement within bound and within 0.5% of its ratio."""
    O = oracle_lib
    g = load_golden(case)
    fields = golden_inputs(g)
    for tag in g["tags"]:
        t = str(tag)
        eb = float(t.split("|")[1])
        res = O.compress(fields, "sz-lcf", "rel", eb, fmt=1)
        assert np.array_equal(res["bounds"], g[f"{t}|bounds"]), t
        for fi in range(6):
            key = f"{t}|payload{fi}_sha"
            if key in g:
                assert sha(res["payloads"][fi]) == str(g[key]), (t, fi)
        assert sha(res["wire"]) == str(g[f"{t}|wire_sha"]), t
        dec = O.decompress(res["wire"])
        for fi in range(6):
            assert sha(dec[fi]) == str(g[f"{t}|recon{fi}_sha"]), (t, fi)
        r2 = O.compress(fields, "sz-lcf", "rel", eb, fmt=2)
        # compressed size never more than 0.5% above the reference's (on
        # escape-heavy noise the dual-quant LCF chain is smaller)
        assert r2["ratio"] >= float(g[f"{t}|ratio"]) * (1 - 0.005), (t, r2["ratio"])
        d2 = O.decompress(r2["wire"])
        for fi in range(6):
            err = np.abs(fields[fi].astype(np.float64) - d2[fi].astype(np.float64))
            assert float(err.max()) <= r2["bounds"][fi] or r2["mask"] & (1 << fi)


# ---------------------------------------------------------------- CPC2000 family

@pytest.mark.parametrize("case", CPC_CASES)
def test_oracle_cpc_matches_reference(oracle_lib, case):
    """sz-cpc2000 / cpc2000: the oracle's fmt-1 archive is the reference's
    byte for byte (full-key sort, raw first key + unsigned VLC deltas per
    segment, per-segment scheme choice, float32 corrections, SZ or signed-VLC
    velocities, segment minima in the container), and decoding the
    reference's archive reproduces the reference's reconstruction exactly."""
    O = oracle_lib
    g = load_golden(case)
    fields = golden_inputs(g)
    ss = int(g["segment_size"])
    for tag in g["tags"]:
        t = str(tag)
        mode, eb = t.split("|")
        if f"{t}|error" in g:
            with pytest.raises(OverflowError):
                O.compress_cpc(fields, mode, "rel", float(eb), segment_size=ss, fmt=1)
            continue
        res = O.compress_cpc(fields, mode, "rel", float(eb), segment_size=ss, fmt=1)
        ref = bytes(g[f"{t}|wire"])
        assert res["wire"] == ref, tag
        assert np.array_equal(res["order"], g[f"{t}|order"]), tag
        out = O.decompress_cpc(ref)
        for fi in range(6):
            assert np.array_equal(out[fi].view(np.uint32), g[f"{t}|recon{fi}"].view(np.uint32)), (tag, fi)


@pytest.mark.parametrize("case", CPC_CASES)
def test_oracle_cpc_v2_roundtrip_and_ratio(oracle_lib, case):
    """fmt 2 (what the GPU writes: per-segment bit lengths appended to every
    VLC-family payload, dual-quant SZ velocities) decodes to the same
    coordinates and VLC velocities as fmt 1, every value within its bound,
    ratio within 0.5% of the reference's (inputs of >= 1000 particles)."""
    O = oracle_lib
    g = load_golden(case)
    fields = golden_inputs(g)
    ss = int(g["segment_size"])
    for tag in g["tags"]:
        t = str(tag)
        if f"{t}|error" in g:
            continue
        mode, eb = t.split("|")
        r2 = O.compress_cpc(fields, mode, "rel", float(eb), segment_size=ss, fmt=2)
        out = O.decompress_cpc(r2["wire"])
        ref = O.decompress_cpc(bytes(g[f"{t}|wire"]))
        order = r2["order"]
        for fi in range(6):
            if fi < 3 or mode == "cpc2000":
                assert np.array_equal(out[fi].view(np.uint32), ref[fi].view(np.uint32)), (tag, fi)
            if r2["mask"] & (1 << fi):
                continue
            err = np.abs(fields[fi][order].astype(np.float64) - out[fi].astype(np.float64))
            assert float(err.max()) <= r2["bounds"][fi], (tag, fi)
        if fields[0].size >= 1000:
            assert abs(r2["ratio"] / float(g[f"{t}|ratio"]) - 1) < 0.005, (tag, r2["ratio"])
