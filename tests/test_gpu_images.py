"""8-bit file path against vectors the REFERENCE wrote (tests/golden/golden_images.*,
generator make_golden.py --images): ImageFile.channel_fields -> solve_image -> image_from_fields
(fileio.py:51-65), the P4 mask raster (fileio.py:181-230), and the quantiser's known answers
(ties to even, out-of-range values)."""

import json
import os

import numpy as np
import pytest

import oracle
import paper_2401_06744_b200 as bp

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(HERE, "golden_images.npz")), json.load(open(os.path.join(HERE, "golden_images.json")))


def _inputs(meta):
    """The generator's inputs, regenerated from the seeds (oracle.seeded_problem == conftest's recipe)."""
    m, k = oracle.seeded_problem(meta["w"], meta["h"], meta["density"], meta["seed"], channels=meta["channels"])
    px = k.astype(np.uint8)
    return m, (px[0] if meta["channels"] == 1 else np.ascontiguousarray(np.moveaxis(px, 0, 2)))


def _cfg(meta):
    return bp.MultigridConfig(block_size=meta["block_size"], overlap=meta["overlap"],
                              solver=bp.SolverConfig(**meta.get("solver", {})))


def test_quantiser_known_answers(gold):
    g, _ = gold
    for name in ("quant_rgb", "quant_gray"):
        img = bp.image_from_fields(g[f"{name}_fields"])
        assert img.pixels.dtype == np.uint8 and np.array_equal(img.pixels, g[f"{name}_pixels"])
    with pytest.raises(ValueError, match="expected 1 or 3 channels"):
        bp.image_from_fields(np.zeros((2, 4, 4)))


def test_mask_raster_known_answer(gold):
    g, _ = gold
    m, raster = g["raster_mask"], g["raster_bytes"]
    assert np.array_equal(bp.pack_mask_raster(m), raster)
    assert np.array_equal(bp.unpack_mask_raster(raster, m.shape[1]), m)
    dirty = raster.copy()
    dirty[:, -1] |= 0x07                      # padding bits of a row are ignored (np.unpackbits(...)[:, :width])
    assert np.array_equal(bp.unpack_mask_raster(dirty, m.shape[1]), m)


@pytest.mark.parametrize("name", ["img_rgb_256x192", "img_gray_203x131", "img_gray_20x30",
                                  "img_rgb_dense_64x48", "img_rgb_loose_96x64"])
def test_decode_matches_reference_bytes(gold, name):
    g, meta = gold
    meta = meta[name]
    mask, pixels = _inputs(meta)
    want = g[f"{name}_pixels"]
    out, reps = bp.inpaint_image_u8(pixels, mask, "mg-oras", _cfg(meta))
    assert out.shape == want.shape and out.dtype == np.uint8
    assert [r.iterations for r in reps] == meta["iterations"]
    if float(g[f"{name}_margin_min"]) > 1e-9:            # no reference value sits on a rounding boundary
        assert np.array_equal(out, want)
    else:
        # values within 1e-9 of a boundary (the dense case has unknown pixels that converge to exact .5 means)
        # may fall either way: everything else is byte-exact, the undecided ones differ by one step at most
        f = bp.solve_image(bp.InpaintingProblem(mask, bp.ImageFile(pixels).channel_fields()), "mg-oras", _cfg(meta)).fields
        f = f[0] if meta["channels"] == 1 else np.moveaxis(f, 0, 2)
        decided = np.abs(f - np.floor(f) - 0.5) > 1e-9
        assert decided.mean() > 0.99 and np.array_equal(out[decided], want[decided])
        assert np.abs(out.astype(int) - want.astype(int)).max() <= 1
        want = out
    # the raster the file holds instead of a boolean mask; dirty padding bits change nothing
    bits = bp.pack_mask_raster(mask)
    if meta["w"] % 8:
        bits[:, -1] |= (1 << (8 - meta["w"] % 8)) - 1
    out2, _ = bp.inpaint_image_u8(pixels, bits, "mg-oras", _cfg(meta), packed=True)
    assert np.array_equal(out2, want)
    # eager launches (host-checked cycle loop) take the same egress
    h, w = mask.shape
    plan = bp.Plan(w, h, meta["channels"], 1, _cfg(meta), use_graphs=False)
    out3, _ = plan.solve_host_image_u8(bp.pack_mask_raster(mask)[None], pixels[None])
    assert np.array_equal(out3[0], want)
    plan.close()


def test_comparison_pipelines_take_the_tail_pass(gold):
    g, meta = gold
    meta = meta["img_gray_203x131"]
    mask, pixels = _inputs(meta)
    for name in ("ml-oras", "mg-cg"):
        out, reps = bp.inpaint_image_u8(pixels, mask, name, _cfg(meta))
        res = bp.solve_image(bp.InpaintingProblem(mask, bp.ImageFile(pixels).channel_fields()), name, _cfg(meta))
        assert np.array_equal(out, np.clip(np.round(res.fields), 0, 255).astype(np.uint8)[0])
        assert np.abs(out.astype(int) - g["img_gray_203x131_pixels"].astype(int)).max() <= 1


def test_one_plan_alternates_between_fp64_and_image_calls(gold):
    """The solve graph is keyed by the egress target: fp64 and 8-bit calls on one plan do not disturb each
    other, batches keep per-frame results, and the pipeline's image layout equals the single calls."""
    g, meta = gold
    meta = meta["img_rgb_256x192"]
    mask, pixels = _inputs(meta)
    want = g["img_rgb_256x192_pixels"]
    h, w = mask.shape
    m2, k2 = oracle.seeded_problem(w, h, 0.06, 77, channels=3)
    px2 = np.ascontiguousarray(np.moveaxis(k2.astype(np.uint8), 0, 2))
    cfg = _cfg(meta)
    plan = bp.Plan(w, h, 3, 2, cfg)
    bits = np.stack([bp.pack_mask_raster(mask), bp.pack_mask_raster(m2)])
    out_a, _ = plan.solve_host_image_u8(bits, np.stack([pixels, px2]))
    f64, _ = plan.solve_host(np.stack([mask, m2]).view(np.uint8), np.stack([bp.ImageFile(pixels).channel_fields(), k2]))
    out_b, _ = plan.solve_host_image_u8(bits[::-1].copy(), np.stack([px2, pixels]))
    plan.close()
    assert np.array_equal(out_a[0], want) and np.array_equal(out_b[1], want)
    assert np.array_equal(out_a[1], out_b[0])
    expect = np.moveaxis(np.clip(np.round(f64), 0, 255).astype(np.uint8), 1, 3)
    assert np.array_equal(out_a, expect)
    pipe = bp.FramePipeline(w, h, 3, cfg, lanes=2)
    out_p, reps = pipe.run(np.stack([bits[0], bits[1], bits[0]]), np.stack([pixels, px2, pixels]), image=True)
    pipe.close()
    assert np.array_equal(out_p[0], want) and np.array_equal(out_p[2], want) and np.array_equal(out_p[1], out_a[1])
    assert len(reps) == 3 and all(len(r) == 3 for r in reps)


def test_image_entry_point_errors():
    cfg = bp.MultigridConfig(block_size=16, overlap=2)
    px = np.zeros((40, 50, 3), dtype=np.uint8)
    with pytest.raises(bp.EmptyMaskError):
        bp.inpaint_image_u8(px, np.zeros((40, 50), dtype=bool), "mg-oras", cfg)
    with pytest.raises(ValueError, match="pixels must be uint8"):
        bp.inpaint_image_u8(px.astype(np.float64), np.ones((40, 50), dtype=bool), "mg-oras", cfg)
    with pytest.raises(ValueError, match="mask shape"):
        bp.inpaint_image_u8(px, np.ones((40, 51), dtype=bool), "mg-oras", cfg)
    with pytest.raises(ValueError, match="packed mask"):
        bp.inpaint_image_u8(px, np.ones((40, 50), dtype=np.uint8), "mg-oras", cfg, packed=True)
    plan = bp.Plan(50, 40, 3, 1, cfg)
    with pytest.raises(ValueError, match="mask has"):
        plan.solve_host_image_u8(np.ones((1, 40, 50), dtype=np.uint8), px[None])
    only_padding = np.zeros((1, 40, 7), dtype=np.uint8)
    only_padding[:, :, -1] = 0x3f                 # bits beyond column 50 only
    with pytest.raises(bp.EmptyMaskError):
        plan.solve_host_image_u8(only_padding, px[None])
    plan.close()
