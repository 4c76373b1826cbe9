#!/usr/bin/env python3
"""Dump golden vectors from the REFERENCE package itself (nbz, read-only at
/root/reference/pkg/src) into tests/golden/.

These fixtures pin the CPU oracle (oracle/) to the reference: the oracle must
reproduce every key, permutation, code, Huffman table, payload and whole v1
archive recorded here byte for byte.  Large arrays are stored as SHA-256
digests; inputs are stored verbatim so the fixtures do not depend on the
generator staying stable.

Run in this container only (the reference does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nbz_numba PYTHONPATH=/root/reference/pkg/src \
        python scripts/make_golden.py
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbz_numba")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

import nbz  # noqa: E402
from nbz import _kernels as K  # noqa: E402
from nbz import encode as E  # noqa: E402
from nbz.model import ErrorBoundSpec, ParticleSnapshot  # noqa: E402
from nbz.pipeline import Mode, Settings, compress, decompress, ratio  # noqa: E402
from nbz.quantize import integerize, quantize_field, quantize_residual  # noqa: E402
from nbz.predict import PredictorKind  # noqa: E402
from nbz.rindex import build_r_indices, prx_sort  # noqa: E402

from paper_1711_03888_b200 import datagen as D  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def h(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(bytes(a)).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dump_case(name: str, fields, modes, ebs, settings=Settings()):
    snap = ParticleSnapshot(*fields)
    rec = {f"in_{i}": np.asarray(f, np.float32) for i, f in enumerate(fields)}
    meta = []
    for mode in modes:
        for eb in ebs:
            tag = f"{mode.value}|{eb:g}"
            res = compress(snap, mode, ErrorBoundSpec.relative(eb), settings)
            ar = res.archive
            wire = ar.serialized()
            rec[f"{tag}|wire_sha"] = np.array(h(wire))
            rec[f"{tag}|wire_len"] = np.array(len(wire))
            rec[f"{tag}|ratio"] = np.array(ratio(ar) if ar.n else -1.0)
            rec[f"{tag}|bounds"] = np.array(ar.bounds, np.float64)
            rec[f"{tag}|mask"] = np.array(ar.constant_mask)
            rec[f"{tag}|seg_bits"] = np.array([s.bits for s in ar.segments], np.uint8)
            if res.order is not None:
                rec[f"{tag}|order_sha"] = np.array(h(res.order.astype(np.int64)))
            work = snap if res.order is None else ParticleSnapshot(
                *(f[res.order] for f in snap.fields()))
            for st in ar.streams:
                fi = st.field
                rec[f"{tag}|payload{fi}_sha"] = np.array(h(st.payload))
                q, _ = quantize_field(work.field(fi), PredictorKind.LV, ar.bounds[fi],
                                      ar.interval_count)
                rec[f"{tag}|codes{fi}_sha"] = np.array(h(q.codes.astype(np.int32)))
                rec[f"{tag}|nesc{fi}"] = np.array(q.escapes.shape[0])
                table = E.huffman_build(np.bincount(q.codes))
                rec[f"{tag}|syms{fi}"] = table.symbols.astype(np.int32)
                rec[f"{tag}|lens{fi}"] = table.lengths.astype(np.uint8)
            if ar.n:
                out = decompress(ar)
                for fi in range(6):
                    rec[f"{tag}|recon{fi}_sha"] = np.array(h(out.field(fi)))
            if mode is Mode.SZ_LV_PRX and ar.n:
                resolved = ar.bounds
                cols = [integerize(snap.field(i), resolved[i]).ints
                        if not ar.is_constant(i) else np.zeros(ar.n, np.int64)
                        for i in range(3)]
                keys, segs = build_r_indices(cols, settings.segment_size)
                rec[f"{tag}|keys_sha"] = np.array(h(keys))
                order = prx_sort(keys, segs, settings.ignored_groups, 3)
                assert np.array_equal(order, res.order)
            meta.append(tag)
    rec["tags"] = np.array(meta)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
    print(name, len(meta), "tags")


def dump_variant_case(name: str, fields, ebs, segment_size: int = 16384, ig: int = 6):
    """R-index variants (rindex.py:24-44): velocity keys, and six-field
    coord+velocity keys (group width 6, 10-bit cap), sz-lv-prx."""
    from nbz.rindex import RIndexVariant
    snap = ParticleSnapshot(*fields)
    rec = {f"in_{i}": np.asarray(f, np.float32) for i, f in enumerate(fields)}
    meta = []
    for variant in (RIndexVariant.VELOCITY, RIndexVariant.COORD_VELOCITY):
        settings = Settings(segment_size=segment_size, ignored_groups=ig, rindex_variant=variant)
        for eb in ebs:
            tag = f"{variant.value}|{eb:g}"
            res = compress(snap, Mode.SZ_LV_PRX, ErrorBoundSpec.relative(eb), settings)
            ar = res.archive
            wire = ar.serialized()
            rec[f"{tag}|wire_sha"] = np.array(h(wire))
            rec[f"{tag}|wire_len"] = np.array(len(wire))
            rec[f"{tag}|ratio"] = np.array(ratio(ar))
            rec[f"{tag}|bounds"] = np.array(ar.bounds, np.float64)
            rec[f"{tag}|mask"] = np.array(ar.constant_mask)
            rec[f"{tag}|seg_bits"] = np.array([sg.bits for sg in ar.segments], np.uint8)
            rec[f"{tag}|order_sha"] = np.array(h(res.order.astype(np.int64)))
            cols = [integerize(snap.field(i), ar.bounds[i]).ints if not ar.is_constant(i)
                    else np.zeros(ar.n, np.int64) for i in variant.field_indices]
            keys, segs = build_r_indices(cols, segment_size)
            rec[f"{tag}|keys_sha"] = np.array(h(keys))
            out = decompress(ar)
            for fi in range(6):
                rec[f"{tag}|recon{fi}_sha"] = np.array(h(out.field(fi)))
            meta.append(tag)
    rec["tags"] = np.array(meta)
    rec["segment_size"] = np.array(segment_size)
    rec["ignored_groups"] = np.array(ig)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
    print(name, len(meta), "tags")


def dump_lcf_case(name: str, fields, ebs):
    """sz-lcf (mode uid 0): the LCF predictor pred = 2*prev - prev2
    (_kernels.py:162-165), no R-index."""
    snap = ParticleSnapshot(*fields)
    rec = {f"in_{i}": np.asarray(f, np.float32) for i, f in enumerate(fields)}
    meta = []
    for eb in ebs:
        tag = f"sz-lcf|{eb:g}"
        res = compress(snap, Mode.SZ_LCF, ErrorBoundSpec.relative(eb))
        ar = res.archive
        wire = ar.serialized()
        rec[f"{tag}|wire_sha"] = np.array(h(wire))
        rec[f"{tag}|wire_len"] = np.array(len(wire))
        rec[f"{tag}|ratio"] = np.array(ratio(ar))
        rec[f"{tag}|bounds"] = np.array(ar.bounds, np.float64)
        rec[f"{tag}|mask"] = np.array(ar.constant_mask)
        for st in ar.streams:
            rec[f"{tag}|payload{st.field}_sha"] = np.array(h(st.payload))
        out = decompress(ar)
        for fi in range(6):
            rec[f"{tag}|recon{fi}_sha"] = np.array(h(out.field(fi)))
        meta.append(tag)
    rec["tags"] = np.array(meta)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
    print(name, len(meta), "tags")


def dump_cpc_case(name: str, fields, ebs, segment_size: int = 16384):
    """CPC2000 family (mode uids 3, 4): the full-key R-index coordinate codec
    (raw first key + unsigned VLC key deltas per segment, float32
    corrections; pipeline.py:316-375, 460-500) with SZ (sz-cpc2000) or
    signed-VLC (cpc2000) velocities.  Whole wires are stored verbatim."""
    snap = ParticleSnapshot(*fields)
    rec = {f"in_{i}": np.asarray(f, np.float32) for i, f in enumerate(fields)}
    meta = []
    settings = Settings(segment_size=segment_size)
    for mode in (Mode.SZ_CPC2000, Mode.CPC2000):
        for eb in ebs:
            tag = f"{mode.value}|{eb:g}"
            try:
                res = compress(snap, mode, ErrorBoundSpec.relative(eb), settings)
            except Exception as exc:  # e.g. BoundTooSmallError (no key clamp)
                rec[f"{tag}|error"] = np.array(type(exc).__name__)
                meta.append(tag)
                continue
            ar = res.archive
            wire = ar.serialized()
            rec[f"{tag}|wire"] = np.frombuffer(wire, np.uint8)
            rec[f"{tag}|ratio"] = np.array(ratio(ar) if ar.n else -1.0)
            rec[f"{tag}|bounds"] = np.array(ar.bounds, np.float64)
            if res.order is not None:
                rec[f"{tag}|order"] = res.order.astype(np.int64)
            if ar.n:
                out = decompress(ar)
                for fi in range(6):
                    rec[f"{tag}|recon{fi}"] = out.field(fi)
            meta.append(tag)
    rec["tags"] = np.array(meta)
    rec["segment_size"] = np.array(segment_size)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
    print(name, len(meta), "tags")


def dump_kats():
    rec = {}
    # interleave field-order KATs (test_rindex.py:23-29 style) and a random sweep
    rng = np.random.default_rng(7)
    x = rng.integers(0, 1 << 21, 1000).astype(np.int64)
    y = rng.integers(0, 1 << 21, 1000).astype(np.int64)
    z = rng.integers(0, 1 << 21, 1000).astype(np.int64)
    keys = np.empty(1000, np.uint64)
    K.interleave3(x, y, z, keys)
    rec["il_x"], rec["il_y"], rec["il_z"], rec["il_keys"] = x, y, z, keys
    # half-even integerize (test_quantize.py:90-97 style) plus exact ties
    xi = np.array([1.0, 2.0, 3.05, 0.25, 0.75, -0.25, -0.75, 1.25, 2.5], np.float32)
    rec["int_x"] = xi
    rec["int_b"] = np.array(0.05)
    rec["int_out"] = integerize(xi, 0.05).ints
    rec["int_x2"] = xi
    rec["int_out2"] = integerize(xi, 0.125).ints
    # quantize_residual KATs (test_quantize.py:13-27)
    qr = [quantize_residual(r, p, b, 65536) for r, p, b in
          [(10.0, 10.0, 0.1), (10.2, 10.0, 0.1), (1e9, 0.0, 1e-3), (-3.3, 1.0, 0.05)]]
    rec["qr_codes"] = np.array([c for c, _ in qr], np.int64)
    rec["qr_recon"] = np.array([r for _, r in qr], np.float64)
    # exact sz chain with forced escapes (test_kernels_equiv.py:14-26 style)
    xs = rng.normal(0, 50, 4000).astype(np.float32)
    xs[::97] *= 1e7
    codes = np.zeros(xs.size, np.int32)
    recon = np.zeros(xs.size, np.float32)
    esc = np.zeros(xs.size, np.float32)
    ne = K.sz_quantize(xs, 0.01, 32768, False, codes, recon, esc)
    rec["szq_x"], rec["szq_codes"], rec["szq_recon"], rec["szq_esc"] = xs, codes.copy(), recon.copy(), esc[:ne].copy()
    ne2 = K.sz_quantize(xs, 0.01, 32768, True, codes, recon, esc)
    rec["szq_lcf_codes"], rec["szq_lcf_esc"] = codes.copy(), esc[:ne2].copy()
    # huffman lengths: random counts and tie-heavy counts
    c1 = np.sort(rng.integers(1, 10 ** 6, 300)).astype(np.int64)
    rec["hl_c1"], rec["hl_l1"] = c1, K.huffman_lengths(c1)
    c2 = np.sort(np.repeat(np.array([1, 1, 2, 3, 5, 5, 5, 8, 8, 13], np.int64), 7))
    rec["hl_c2"], rec["hl_l2"] = c2, K.huffman_lengths(c2)
    c3 = np.array([4], np.int64)
    rec["hl_c3"], rec["hl_l3"] = c3, K.huffman_lengths(c3)
    # huffman_build on a bincount with ties, and its encode/decode
    syms = rng.integers(0, 200, 20000).astype(np.int32)
    hist = np.bincount(syms)
    table = E.huffman_build(hist)
    bs = E.huffman_encode(syms, table)
    rec["hb_syms_in"] = syms
    rec["hb_symbols"], rec["hb_lengths"] = table.symbols, table.lengths
    rec["hb_bytes"] = np.frombuffer(bs.to_bytes(), np.uint8)
    rec["hb_bits"] = np.array(bs.bit_length)
    # crc64 check value (test_kernels_equiv.py:164-165) and a long buffer
    rec["crc_123456789"] = np.array(K.crc64(b"123456789"), np.uint64)
    buf = rng.integers(0, 256, 100003).astype(np.uint8)
    rec["crc_buf"], rec["crc_buf_val"] = buf, np.array(K.crc64(buf.tobytes()), np.uint64)
    np.savez_compressed(os.path.join(OUT, "kats.npz"), **rec)
    print("kats")


def main():
    os.makedirs(OUT, exist_ok=True)
    K.warmup()
    if "--lcf" in sys.argv:  # only the sz-lcf fixtures
        dump_lcf_case("lcf_hacc24", D.small_hacc(24), [1e-3, 1e-4])
        rng = np.random.default_rng(11)
        noise = [rng.uniform(0, 100, 20000).astype(np.float32) for _ in range(3)]
        noise += [(rng.standard_cauchy(20000) * 10).astype(np.float32) for _ in range(3)]
        dump_lcf_case("lcf_noise20k", noise, [1e-4, 1e-6])
        return
    if "--cpc" in sys.argv:  # only the CPC2000-family fixtures
        dump_cpc_case("cpc_hacc24", D.small_hacc(24), [1e-3, 1e-4])
        dump_cpc_case("cpc_amdf20k", D.small_amdf(20000), [1e-4, 1e-5], segment_size=4096)
        rng = np.random.default_rng(31)
        cst = [rng.uniform(0, 100, 5000).astype(np.float32) for _ in range(6)]
        cst[1] = np.full(5000, 7.25, np.float32)
        cst[4] = np.full(5000, -3.5, np.float32)
        dump_cpc_case("cpc_const2", cst, [1e-4], segment_size=1000)
        noise = [rng.uniform(0, 100, 9000).astype(np.float32) for _ in range(3)]
        noise += [(rng.standard_cauchy(9000) * 10).astype(np.float32) for _ in range(3)]
        dump_cpc_case("cpc_noise9k", noise, [1e-4, 1e-6], segment_size=2048)
        dump_cpc_case("cpc_tiny", [rng.uniform(0, 10, 3).astype(np.float32) for _ in range(6)],
                      [1e-4])
        return
    if "--variants" in sys.argv:  # only the R-index variant fixtures
        dump_variant_case("variants_hacc24", D.small_hacc(24), [1e-3, 1e-4])
        dump_variant_case("variants_amdf20k", D.small_amdf(20000), [1e-4], segment_size=4096, ig=2)
        return
    dump_kats()
    both = [Mode.SZ_LV, Mode.SZ_LV_PRX]
    dump_case("hacc34", D.small_hacc(34), both, [1e-4])
    dump_case("amdf40k", D.small_amdf(40000), both, [1e-4])
    dump_case("sweep_hacc20", D.small_hacc(20), both, [1e-2, 1e-3, 1e-5, 1e-6])
    dump_case("sweep_amdf8k", D.small_amdf(8000), both, [1e-2, 1e-3, 1e-5, 1e-6])
    rng = np.random.default_rng(20260808)
    # edge cases: tiny, constant field, escape-heavy noise, single segment
    dump_case("tiny1", [np.array([1.5], np.float32)] * 6, both, [1e-4])
    t3 = [rng.uniform(0, 10, 3).astype(np.float32) for _ in range(6)]
    dump_case("tiny3", t3, both, [1e-4])
    cst = [rng.uniform(0, 100, 5000).astype(np.float32) for _ in range(6)]
    cst[1] = np.full(5000, 7.25, np.float32)
    cst[4] = np.full(5000, -3.5, np.float32)
    dump_case("const2", cst, both, [1e-4])
    noise = [rng.uniform(0, 100, 20000).astype(np.float32) for _ in range(3)]
    noise += [(rng.standard_cauchy(20000) * 10).astype(np.float32) for _ in range(3)]
    dump_case("noise20k", noise, both, [1e-4, 1e-6])
    print("done")


if __name__ == "__main__":
    main()
