"""CPU tests: the C ABI loads and exports every declared symbol; host-side
integer ports (stream ids, sign masks) agree with the oracle; API validation
that needs no device."""

import os
import re

import numpy as np
import pytest

from oracle import nvfp4_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    from paper_2601_22813_b200 import _lib
    header = open(os.path.join(ROOT, "include", "quartet2.h")).read()
    declared = set(re.findall(r"\b(q2_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    lib = _lib.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.q2_version().startswith(b"quartet2-b200")


def test_sf_bytes():
    from paper_2601_22813_b200 import _lib
    L = _lib.lib()
    assert L.q2_sf_bytes(128, 64) == 1024
    assert L.q2_sf_bytes(257, 64) == 2048
    assert L.q2_sf_bytes(128, 256) == 4096
    assert L.q2_sf_bytes(256, 80) == 2 * 1024


def test_host_streams_match_oracle():
    import paper_2601_22813_b200 as q2
    for parts in [(1,), (2,), ("mse-data", 0), (q2.PAIR_DX, 0), (q2.PAIR_DW, 1), (2**64 - 1, 5)]:
        assert q2.derive_stream(*parts) == O.derive_stream(*parts)
    for seed, rot in [(0, q2.PAIR_DX), (7, q2.PAIR_DW), (2**63 + 5, 3)]:
        w = q2.sign_mask(seed, rot)
        assert sum(v << (32 * i) for i, v in enumerate(w)) == O.sign_mask(seed, rot)
    for idx in (0, 1, 12345, 2**40):
        assert q2.prng_uniform(9, 77, idx) == float(O.prng_uniform(9, 77, idx))


def test_sf_layout_formula():
    """The scale layout (include/quartet2.h) is a bijection onto the 1 KiB blocks,
    and per block half (the source of one tcgen05.cp.32x128b.warpx4) TMEM lane L
    / column c holds the scale of row 128*half + 32*c + L (the tcgen05
    block-scale vector layout; one K=64 MMA block per 1 KiB)."""
    def off(r, j, K):
        kb = (K + 63) // 64
        L = r % 32
        return (((r // 256) * kb + j // 4) * 1024 + (L // 8) * 256 + ((r // 128) % 2) * 128 + (L % 8) * 16
                + ((r % 128) // 32) * 4 + j % 4)
    K, R = 256, 512
    seen = {off(r, j, K) for r in range(R) for j in range(K // 16)}
    assert len(seen) == R * K // 16 and max(seen) < R * K // 16
    def lane_col(b):                       # block byte -> (half, lane, column, byte-in-column)
        g, rest = divmod(b % 1024, 256)
        half, rest = divmod(rest, 128)
        row8, byte = divmod(rest, 16)
        return half, 8 * g + row8, byte // 4, byte % 4
    for r in (0, 5, 37, 100, 127, 128, 200, 255, 300):
        for j in (0, 3, 4, 7, 13):
            half, lane, col, i = lane_col(off(r, j, K))
            assert r % 256 == 128 * half + 32 * col + lane and i == j % 4
            assert off(r, j, K) // 1024 == (r // 256) * (K // 64) + j // 4


def test_layer_config_validation():
    import paper_2601_22813_b200 as q2
    with pytest.raises(ValueError):
        q2.LayerConfig(forward_scheme="rtn_32x32")
    with pytest.raises(ValueError):
        q2.LayerConfig(reuse_forward_weights=True)                  # ms_eden re-quantizes W
    with pytest.raises(ValueError):
        q2.LayerConfig("rtn_1x16", "sr_rht", reuse_forward_weights=True)   # dense reused W^T: not built
    with pytest.raises(ValueError):
        q2.LayerConfig(backward_scheme="sr_rtn")
    with pytest.raises(ValueError):
        q2.baseline_config("quartet3")
    assert q2.baseline_config("identity") == q2.LayerConfig("identity", "identity")
    assert q2.baseline_config("four_over_six_backward").backward_scheme == "sr_46"
    assert q2.baseline_config("quartet2") == q2.LayerConfig()
    assert q2.baseline_config("tetrajet_v2") == q2.LayerConfig("rtn_1x16", "sr_rht")
    assert q2.baseline_config("nvidia") == q2.LayerConfig("rtn_16x16", "sr_rht", reuse_forward_weights=True)
    assert q2.baseline_config("four_over_six").forward_scheme == "rtn_16x16_46"


def test_constants_match_reference_arithmetic():
    import paper_2601_22813_b200 as q2
    assert (6.0 * q2.GUARDED_SCALE_CAP).hex() == "0x1.3c3c3c3c3c3c4p+11"
    from paper_2601_22813_b200.rht import INV_SQRT_CHUNK
    assert INV_SQRT_CHUNK.hex() == "0x1.6a09e667f3bcdp-4"


def test_module_host_side():
    import torch
    import paper_2601_22813_b200 as q2
    m = q2.Quartet2Linear(256, 128, bias=True, seed=5)
    assert m.weight.shape == (128, 256) and m.weight.dtype == torch.bfloat16 and m.bias.shape == (128,)
    assert m.seeds_for(3) == q2.SeedPair(q2.derive_stream(5, 1, 3), q2.derive_stream(5, 2, 3))
    assert m.seeds_for(0) != q2.Quartet2Linear(256, 128, seed=6).seeds_for(0)
    assert "posthoc=False" in repr(m) and m.cfg == q2.baseline_config("quartet2")


def test_ablation_config_validation():
    import paper_2601_22813_b200 as q2
    for abl in q2.ABLATIONS:
        q2.LayerConfig("rtn_1x16", "sr_rht", ablation=abl)
    for abl in ("b", "d"):
        with pytest.raises(ValueError, match="ms_eden cannot quantize a single GEMM operand"):
            q2.LayerConfig(ablation=abl)
    q2.LayerConfig(ablation="a"), q2.LayerConfig(ablation="c")
    with pytest.raises(ValueError, match="unknown ablation"):
        q2.LayerConfig(ablation="f")
    with pytest.raises(ValueError, match="weight reuse requires a square-block forward scheme"):
        q2.LayerConfig("rtn_1x16", "sr", reuse_forward_weights=True)
    with pytest.raises(ValueError, match=r"known: \['four_over_six', 'four_over_six_backward', 'identity'"):
        q2.baseline_config("quartet3")


def test_config_text_round_trip():
    import paper_2601_22813_b200 as q2
    for name in ("quartet2", "nvidia", "four_over_six_backward", "identity"):
        cfg = q2.baseline_config(name)
        assert q2.parse_config(q2.format_config(cfg)) == cfg
    cfg = q2.LayerConfig("rtn_1x16", "sr_rht", ablation="d", posthoc=True)
    assert q2.parse_config(q2.format_config(cfg)) == cfg
    assert q2.format_config(q2.baseline_config("nvidia")) == (
        "forward_scheme = rtn_16x16\nbackward_scheme = sr_rht\nablation = full\nreuse_forward_weights = true\n")
    assert q2.parse_config("# comment\n\nbackward_scheme = sr  # trailing\n") == q2.LayerConfig("identity", "sr")
    for bad, msg in (("forward_scheme", "config line 1: expected key = value"),
                     ("colour = red", "config line 1: unknown key 'colour'"),
                     ("\nreuse_forward_weights = yes", "config line 2: expected true/false")):
        with pytest.raises(ValueError, match=msg):
            q2.parse_config(bad)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted (GPU box)")
def test_config_text_matches_live_reference(tmp_path):
    import sys
    os.environ.setdefault("NUMBA_CACHE_DIR", str(tmp_path))
    sys.path.insert(0, "/root/reference/pkg/src")
    from nvfp4emu import linear_graph as LG
    import paper_2601_22813_b200 as q2
    for name in ("quartet2", "tetrajet_v2", "nvidia", "four_over_six", "four_over_six_backward", "identity"):
        ref = LG.baseline_config(name)
        assert q2.format_config(q2.baseline_config(name)) == LG.format_config(ref)
        ours = q2.parse_config(LG.format_config(ref))
        assert (ours.forward_scheme, ours.backward_scheme, ours.ablation, ours.reuse_forward_weights) == \
            (ref.forward_scheme, ref.backward_scheme, ref.ablation, ref.reuse_forward_weights)
    for text in ("ablation = b", "ablation = b\nbackward_scheme = sr", "reuse_forward_weights = true",
                 "forward_scheme = rtn_16x16\nbackward_scheme = ms_eden\nreuse_forward_weights = true"):
        outcomes = []
        for parse in (LG.parse_config, q2.parse_config):
            try:
                c = parse(text)
                outcomes.append((c.forward_scheme, c.backward_scheme, c.ablation, c.reuse_forward_weights))
            except ValueError as exc:
                outcomes.append(str(exc))
        assert outcomes[0] == outcomes[1], (text, outcomes)

def test_reports_to_json_stable():
    import json
    import numpy as np
    from paper_2601_22813_b200 import harness as H
    r = H.MseReport("quartet2", "1x16", np.float64(1.5e-3), 1e-6, 1000, 0)
    text = H.reports_to_json({"mse": [r], "slope": np.float32(-1.0), "b": np.arange(3)})
    assert text == H.reports_to_json({"b": np.arange(3), "slope": np.float32(-1.0), "mse": [r]})
    d = json.loads(text)
    assert d["mse"][0]["mse_e3"] == 1.5 and d["b"] == [0, 1, 2] and text.endswith("\n")
    with pytest.raises(TypeError, match="not JSON-serializable"):
        H.reports_to_json({"x": object()})


def test_custom_ops_fake_shapes():
    """torch.ops.quartet2.* propagate shapes through FakeTensorMode (no GPU needed):
    the whole layer written with the custom ops traces to Y [T, out], dX [T, in], dW [out, in]."""
    import torch
    from torch._subclasses.fake_tensor import FakeTensorMode
    import paper_2601_22813_b200 as q2
    with FakeTensorMode():
        x = torch.empty(256, 512, dtype=torch.bfloat16, device="cuda")
        w = torch.empty(384, 512, dtype=torch.bfloat16, device="cuda")
        e = torch.empty(256, 384, dtype=torch.bfloat16, device="cuda")
        codes, sf, scale = torch.ops.quartet2.quantize_rtn_46(x)
        assert codes.shape == (256, 256) and sf.shape == (q2.ops.sf_bytes(256, 512),) and scale.shape == (1,)
        y, dx, dw = q2.ops.linear_fwd_bwd(x, w, e, q2.SeedPair(1, 2))
        assert (y.shape, dx.shape, dw.shape) == ((256, 384), (256, 512), (384, 512))
        assert y.dtype == torch.bfloat16 and dx.dtype == dw.dtype == torch.float32
    L = q2._lib.lib()
    for R, K in ((256, 512), (300, 80), (16384, 11264)):
        assert q2.ops.sf_bytes(R, K) == L.q2_sf_bytes(R, K)
