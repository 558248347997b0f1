"""Error behaviour and edge cases of the C-ABI, mirroring volprim::Error (errors.h:11-38)."""
import numpy as np
import pytest

from paper_2103_01954_b200 import Renderer, api, synthetic

pytestmark = pytest.mark.gpu


def test_usage_errors(renderer):
    tr, pay = synthetic.shell_arrays(16, 4)
    bad = tr.copy()
    bad[3, 21] = -1.0  # composed scale <= 0 (primitive.cpp:44-45)
    with pytest.raises(api.Error) as e:
        api.compose(bad)
    assert e.value.category == api.ErrorCategory.USAGE and e.value.exit_code == 2
    scene = synthetic.make_shell_scene(16, 4)
    with pytest.raises(api.Error) as e:
        renderer.set_frame(scene, 1)  # march.cpp:96-97
    assert e.value.category == api.ErrorCategory.USAGE
    renderer.set_frame(scene, 0)
    cam = synthetic.shell_camera(-1, 0, 32)
    for cfg in (api.MarchConfig(step_size=0.0), api.MarchConfig(step_size=-1e-3),
                api.MarchConfig(accumulation_permutation=3)):
        with pytest.raises(api.Error) as e:
            renderer.render(cam, cfg)
        assert e.value.category == api.ErrorCategory.USAGE
    xf = api.compose(tr)
    xf[2, 12] = 0.0
    with pytest.raises(api.Error) as e:
        renderer.set_scene_composed(xf, api.PrimitiveSlab(16, 4, pay), api.WindowParams())
    assert e.value.category == api.ErrorCategory.USAGE


def test_render_without_scene_is_usage_error():
    with Renderer(0) as r:
        with pytest.raises(api.Error) as e:
            r.render(synthetic.shell_camera(-1, 0, 16), api.MarchConfig())
        assert e.value.category == api.ErrorCategory.USAGE


def test_empty_scene_and_empty_image(renderer):
    renderer.set_scene_composed(np.zeros((0, 15), np.float32), api.PrimitiveSlab(0, 4, np.zeros(0, np.float32)),
                                api.WindowParams())
    out = renderer.render(synthetic.shell_camera(-1, 0, 48), api.MarchConfig())
    assert out.color.shape == (48, 48, 3) and not out.color.any() and not out.alpha.any()
    assert out.total_samples() == 0
    tr, pay = synthetic.shell_arrays(16, 4)
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(16, 4, pay), api.WindowParams())
    cam = synthetic.shell_camera(-1, 0, 16)
    cam.width = 0
    out = renderer.render(cam, api.MarchConfig())
    assert out.color.size == 0


def test_module_level_render_and_composite():
    scene = synthetic.make_shell_scene(64, 8)
    cam = synthetic.shell_camera(-1, 0, 64)
    out = api.render(scene, 0, cam, api.MarchConfig())
    assert out.color.shape == (64, 64, 3) and out.total_samples() > 0
    bg = np.full((64, 64, 3), 0.25, np.float32)
    img = api.composite(out, bg)
    a = out.alpha
    assert np.allclose(img, a * out.color + (1 - a) * bg, atol=1e-7)


def test_reference_dropin_adapter_is_bitwise_identical():
    """oracle/_ref/dropin_check: the reference's volprim::render vs volprim::render_b200 (the
    adapter of INTEGRATION.md over libvpb.so) on the same Scene, compared bitwise. The binary
    is built where /root/reference exists (oracle/Makefile `dropin`) and travels prebuilt."""
    import pathlib
    import subprocess
    exe = pathlib.Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "dropin_check"
    if not exe.exists():
        pytest.skip("dropin_check not built (needs /root/reference at build time)")
    for args in (["64", "16", "256"], ["512", "8", "384"]):
        r = subprocess.run([str(exe), *args], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "IDENTICAL" in r.stdout
