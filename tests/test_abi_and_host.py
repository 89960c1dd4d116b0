"""CPU: the C-ABI library loads and exports every declared symbol; host-side
logic (synthetic workload, formats, view/row sharding, error mapping) without
touching a GPU."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    hdr = (ROOT / "include" / "semsplat_b200.h").read_text()
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", hdr)) - {"ss_status"})


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2505_08124_b200._lib import LIB_PATH, lib
    lib()  # binds every signature
    so = ctypes.CDLL(str(LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(so, s)]
    assert not missing, missing
    assert len(declared_symbols()) >= 25


def test_library_is_sm100a_only():
    import subprocess
    from paper_2505_08124_b200._lib import LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB_PATH)], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2505_08124_b200 import DeviceError
    from paper_2505_08124_b200._lib import Context
    with pytest.raises(DeviceError):
        Context(0)


def test_synth_embedding_matches_reference_golden():
    from harness.workload import synth_embedding
    from tests.goldens import golden
    z = golden("synth")
    for label, vec in zip(z["labels"], z["vectors"]):
        assert synth_embedding(str(label), 512).tobytes() == vec.tobytes()


def test_mt19937_64_known_answer():
    """std::mt19937_64 default seed: the 10000th output is 9981545732273789042
    (C++11 [rand.predef]); the first is 14514284786278117030."""
    from tests.util import MT19937_64
    m = MT19937_64(5489)
    assert m() == 14514284786278117030
    for _ in range(9998):
        m()
    assert m() == 9981545732273789042


def test_query_store_generator_matches_cmd_bench():
    """main.cpp:440-450: store rows then queries, f32((rng()>>11)+0.5)*2^-53-0.5,
    from std::mt19937_64(seed ^ 0xbe9c)."""
    from harness.workload import query_workload
    from tests.util import MT19937_64
    rows, queries = query_workload(2505, 5, 3, 16)
    m = MT19937_64(2505 ^ 0xBE9C)
    exp = np.array([np.float32(((m() >> 11) + 0.5) * 2.0 ** -53 - 0.5) for _ in range(8 * 16)], np.float32)
    assert rows.shape == (5, 16) and queries.shape == (3, 16)
    assert np.concatenate([rows.ravel(), queries.ravel()]).tobytes() == exp.tobytes()


def test_look_at_matches_reference(ref):
    from harness.workload import orbit_camera
    for v in (0, 7, 333):
        c = orbit_camera(v, 1000, 1152, 864)
        import math
        th = 2 * math.pi * v / 1000
        r = ref.look_at([2 * math.cos(th), 2 * math.sin(th), 16.0], [0, 0, 0], 1152, 864, 0.9 * 1152)
        assert c.rotation.tobytes() == r.rotation.tobytes() and c.translation.tobytes() == r.translation.tobytes()


def test_rect_masks_decode_to_rectangles(oracle):
    from paper_2505_08124_b200.formats import rle_runs_from_bitmap
    from harness.workload import rect_masks
    runs, offs = rect_masks(99, 120, 90, 40)
    assert offs.shape[0] == 41
    for j in range(40):
        r = runs[int(offs[j]):int(offs[j + 1])]
        bits = oracle.rle_decode(r, 120, 90).reshape(90, 120)
        ys, xs = np.nonzero(bits)
        assert bits[ys.min():ys.max() + 1, xs.min():xs.max() + 1].all()  # a filled rectangle
        assert np.array_equal(rle_runs_from_bitmap(bits), r)  # canonical rle_encode stream


def test_formats_roundtrip_reference_fixture(ref, tmp_path):
    from paper_2505_08124_b200 import formats
    mp = ref.write_fixture(str(tmp_path / "fx"), objects=2, per_object=10, views=3, resolution=24, mask_scale=2,
                           dim=8, seed=21)
    man = formats.load_manifest(mp)
    assert man.mask_width == 48 and man.raster_width == 24 and len(man.images) == 3
    a = formats.load_scene_arrays(man.resolve("scene.ply"))
    b = ref.load_scene(man.resolve("scene.ply"))
    assert all(x.tobytes() == y.tobytes() for x, y in zip(a, b))
    cams = formats.load_cameras(man.resolve(man.camera_file))
    rc = ref.load_cameras(man.resolve(man.camera_file))
    assert all(c.rotation.tobytes() == r.rotation.tobytes() and c.fx == r.fx for c, r in zip(cams, rc))
    mr = formats.load_maskset_runs(man.resolve(man.images[0].mask_path), 0)
    formats.save_maskset_runs(mr, str(tmp_path / "m.rle"))
    assert (tmp_path / "m.rle").read_bytes() == Path(man.resolve(man.images[0].mask_path)).read_bytes()
    emb = formats.load_mask_embeddings(man.resolve(man.images[0].embedding_path), 8, mr.n_masks)
    formats.save_mask_embeddings(emb, str(tmp_path / "e.emb"))
    assert (tmp_path / "e.emb").read_bytes() == Path(man.resolve(man.images[0].embedding_path)).read_bytes()
    formats.save_cameras(cams, str(tmp_path / "c.txt"))
    back = formats.load_cameras(str(tmp_path / "c.txt"))
    assert all(x.translation.tobytes() == y.translation.tobytes() for x, y in zip(back, cams))


def test_format_errors():
    from paper_2505_08124_b200 import DataError, FormatError, IoError, formats
    with pytest.raises(IoError):
        formats.load_manifest("/nonexistent/manifest.txt")
    import tempfile
    d = Path(tempfile.mkdtemp())
    (d / "bad.rle").write_bytes(b"nope" * 8)
    with pytest.raises(FormatError):
        formats.load_maskset_runs(str(d / "bad.rle"), 0)
    e = np.ones((2, 4), np.float32)
    formats.save_mask_embeddings(e, str(d / "e.emb"))
    with pytest.raises(DataError):
        formats.load_mask_embeddings(str(d / "e.emb"), 8)
    (d / "m.txt").write_text("version = 1\nbogus = 3\n")
    with pytest.raises(FormatError):
        formats.load_manifest(str(d / "m.txt"))


def test_shard_views_matches_reference_assignment():
    from paper_2505_08124_b200.multigpu import shard_views
    for n, w in ((10, 3), (1000, 8), (7, 8), (0, 2)):
        rr = [shard_views(n, w, r) for r in range(w)]
        assert sorted(sum(rr, [])) == list(range(n))
        assert all(v % w == r for r in range(w) for v in rr[r])
        cc = [shard_views(n, w, r, contiguous=True) for r in range(w)]
        assert sum(cc, []) == list(range(n))


@pytest.mark.parametrize("n,w,blk", [(2_000_000, 8, 0), (2_000_000, 8, 65536), (1501, 2, 97), (7, 8, 0), (5, 3, 2),
                                     (1, 1, 0), (100, 1, 30)])
def test_combine_layout_matches_library(n, w, blk):
    """The Python mirror (multigpu.combine_layout / rows_of) of the library's
    block-cyclic combine layout (ss_combine_layout_for, no device needed):
    every table row is held by exactly one rank, rounds cover rows_alloc."""
    import ctypes as C
    from paper_2505_08124_b200._lib import lib
    from paper_2505_08124_b200.multigpu import combine_layout, rows_of
    ra, br, rd = C.c_uint64(), C.c_uint64(), C.c_uint64()
    assert lib().ss_combine_layout_for(n, w, blk, C.byref(ra), C.byref(br), C.byref(rd)) == 0
    lay = combine_layout(n, w, blk)
    assert (lay["rows_alloc"], lay["block_rows"], lay["rounds"]) == (ra.value, br.value, rd.value)
    held = np.concatenate([rows_of(n, w, r, blk) for r in range(w)])
    assert held.size == lay["rows_alloc"] and np.array_equal(np.sort(held), np.arange(lay["rows_alloc"]))
    assert lay["rows_alloc"] >= n


def test_error_kinds_map_to_reference_exceptions():
    from paper_2505_08124_b200 import errors
    for kind, cls in ((1, errors.ContractError), (2, errors.DataError), (3, errors.NumericError),
                      (4, errors.FormatError), (5, errors.IoError), (6, errors.PipelineError), (7, errors.DeviceError)):
        with pytest.raises(cls):
            errors.raise_for(kind, "x")


def test_encode_scene_contract_errors_before_device():
    from paper_2505_08124_b200 import ContractError, DataError
    from paper_2505_08124_b200.formats import DatasetManifest
    from paper_2505_08124_b200.semsplat import encode_scene
    with pytest.raises(ContractError):
        encode_scene(None, DatasetManifest(raster_width=4, raster_height=4), 0, 0)
    with pytest.raises(DataError):
        encode_scene(None, DatasetManifest(), 1, 0)


def test_library_has_no_unresolved_internal_symbols():
    """Every ss:: function the library calls is defined in it (a missing
    definition would only surface at the first call on a GPU box)."""
    import shutil
    import subprocess
    from paper_2505_08124_b200._lib import LIB_PATH
    nm = shutil.which("nm")
    if nm is None:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-D", "--undefined-only", str(LIB_PATH)], capture_output=True, text=True).stdout
    missing = [line.split()[-1] for line in out.splitlines() if line.split() and line.split()[-1].startswith("_ZN2ss")]
    assert not missing, missing
