"""Engine-level artefacts on the GPU: a scene loaded from a JSON document
with an OBJ mesh runs bit-exact against the reference loading the same document, and the
engine's PHM1 photon dump is byte-identical to the reference's write_photon_dump."""
import numpy as np
import pytest

from paper_2111_06906_b200 import pathreuse as pr
from tests.helpers import compare_state, counts
from tests.test_io import DOC, OBJ_TEXT


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["naive", "error"])
def test_loaded_scene_frames_and_dump(tmp_path, mode):
    from oracle import ref

    (tmp_path / "part.obj").write_text(OBJ_TEXT)
    (tmp_path / "scene.json").write_text(DOC)
    gscene = pr.Scene.load(str(tmp_path / "scene.json"))
    rscene = ref.RefScene.from_text(DOC, str(tmp_path))
    cfg = dict(mode=mode, paths=3000, bounces=5, dm=[2, 2, 8, 8], threshold=0.001, seed=9)
    gpu = pr.Engine(gscene, pr.make_config(**cfg))
    cpu = ref.RefEngine(rscene, pr.make_config(**cfg))
    cpu.set_workers(0)
    n_lights = gpu.info().n_lights
    for f in range(4):
        sg, sc = gpu.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(sc), f"frame {f}"
        bad = compare_state(gpu, cpu, n_lights)
        assert all(v == 0 for v in bad.values()), f"frame {f}: {bad}"
    gpu.write_photon_dump(str(tmp_path / "gpu.phm"))
    cpu.write_photon_dump(str(tmp_path / "ref.phm"))
    assert (tmp_path / "gpu.phm").read_bytes() == (tmp_path / "ref.phm").read_bytes()
    n, b, rec = pr.read_photon_dump(str(tmp_path / "gpu.phm"))
    assert (n, b) == (3000, 5)
    assert np.array_equal(rec.view(np.uint8), gpu.photon_map().view(np.uint8))
    # the image written from the ordered gather equals the reference's writer on its gather
    img = gpu.splat(radius=0.25)
    pr.write_image(img, str(tmp_path / "gpu.ppm"))
    ref.write_image(cpu.gather(radius=0.25)[0], str(tmp_path / "ref.ppm"))
    assert (tmp_path / "gpu.ppm").read_bytes() == (tmp_path / "ref.ppm").read_bytes()
