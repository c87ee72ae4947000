"""GVOL streaming (rb_set_field_gvol).

The file is read in z-slabs through pinned buffers and the GriddedField ctor
runs on device; the result must be the reference's grid bit for bit (same
images / hits as packing the reference's own nodes), for any slab size, and
the errors must be load_density_volume's (scene.cpp:212-240)."""
import numpy as np
import pytest

from golden_io import load

pytestmark = pytest.mark.gpu


def _v(v):
    return (v.x, v.y, v.z)


def _grid(name):
    from paper_1812_05902_b200.scene import DensityGrid
    scene, field, g = load(name)
    grid = DensityGrid(field.nx, field.ny, field.nz, field.origin, field.spacing,
                       g["field_rho"], float(g["field_k"]))
    return scene, field, grid


@pytest.mark.parametrize("name", ["field3d", "shock_particles"])
@pytest.mark.parametrize("slab_planes", [1, 5, 0])
def test_gvol_stream_builds_the_reference_grid(tracer, tmp_path, name, slab_planes):
    from paper_1812_05902_b200 import setup as S
    scene, field, grid = _grid(name)
    path = str(tmp_path / f"{name}.gvol")
    S.save_gvol(grid, path)
    tracer.set_field(field)  # the reference's own nodes
    a = tracer.run_trace(scene, True, True)
    tracer.set_field(None)
    d = tracer.set_field_gvol(path, grid.gladstone_dale,
                              slab_bytes=slab_planes * grid.nx * grid.ny * 4)
    assert (d.nx, d.ny, d.nz) == (grid.nx, grid.ny, grid.nz)
    assert _v(d.origin) == tuple(grid.origin) and _v(d.spacing) == tuple(grid.spacing)
    b = tracer.run_trace(scene, True, True)
    assert np.array_equal(a.image, b.image)
    assert np.array_equal(a.hit_sum, b.hit_sum)
    assert np.array_equal(a.landed, b.landed)


def test_gvol_recentre_matches_build_medium_volume(tracer, tmp_path):
    from paper_1812_05902_b200 import setup as S
    from paper_1812_05902_b200.scene import DensityGrid
    _, _, grid = _grid("field3d")
    shifted = DensityGrid(grid.nx, grid.ny, grid.nz, (0.01, -0.02, 0.3), grid.spacing, grid.rho,
                          grid.gladstone_dale)
    path = str(tmp_path / "v.gvol")
    S.save_gvol(shifted, path)
    c = S.ExperimentConfig()
    c.medium = {"type": "gvol", "path": path}
    c.z_dot_to_volume = 0.05
    want = S.build_medium_volume(c)  # the Python mirror of engine.cpp:27-37
    d = tracer.set_field_gvol(path, grid.gladstone_dale, z_center=c.z_dot_to_volume)
    assert _v(d.origin) == tuple(want.origin)


def _write(path, header: bytes, data: np.ndarray):
    with open(path, "wb") as f:
        f.write(header)
        f.write(np.ascontiguousarray(data, dtype="<f4").tobytes())


@pytest.mark.parametrize("case,msg", [
    ("missing", "load_density_volume: cannot open"),
    ("empty", "load_density_volume: missing header"),
    ("magic", "load_density_volume: malformed GVOL header"),
    ("short_header", "load_density_volume: malformed GVOL header"),
    ("dims", "load_density_volume: invalid dims/spacing"),
    ("spacing", "load_density_volume: invalid dims/spacing"),
    ("truncated", "load_density_volume: truncated data"),
    ("negative", "DensityVolume: densities must be finite and >= 0"),
    ("nan", "DensityVolume: densities must be finite and >= 0"),
    ("k", "gladstone_dale: K must be positive"),
])
def test_gvol_errors_are_the_references(tracer, tmp_path, case, msg):
    path = str(tmp_path / "e.gvol")
    ok_header = b"GVOL1 4 3 5 0.001 0.001 0.002 0 0 0\n"
    rho = np.full(60, 1.2, dtype=np.float32)
    k = 2.26e-4
    if case == "missing":
        path = str(tmp_path / "does_not_exist.gvol")
    elif case == "empty":
        _write(path, b"", rho[:0])
    elif case == "magic":
        _write(path, ok_header.replace(b"GVOL1", b"GVOL2"), rho)
    elif case == "short_header":
        _write(path, b"GVOL1 4 3 5 0.001 0.001\n", rho)
    elif case == "dims":
        _write(path, ok_header.replace(b" 3 ", b" 1 "), rho)
    elif case == "spacing":
        _write(path, ok_header.replace(b"0.002", b"-0.002"), rho)
    elif case == "truncated":
        _write(path, ok_header, rho[:59])
    elif case == "negative":
        rho[17] = -1.0
        _write(path, ok_header, rho)
    elif case == "nan":
        rho[59] = np.nan
        _write(path, ok_header, rho)
    else:
        _write(path, ok_header, rho)
        k = 0.0
    with pytest.raises(Exception, match=msg):
        tracer.set_field_gvol(path, k, slab_bytes=4 * 12)


def test_gvol_truncation_is_reported_before_bad_values(tracer, tmp_path):
    """The reference reads everything, then validates: a truncated file with a
    negative density reports the truncation."""
    path = str(tmp_path / "t.gvol")
    rho = np.full(59, 1.2, dtype=np.float32)
    rho[0] = -1.0
    _write(path, b"GVOL1 4 3 5 0.001 0.001 0.002 0 0 0\n", rho)
    with pytest.raises(Exception, match="truncated data"):
        tracer.set_field_gvol(path, 2.26e-4, slab_bytes=4 * 12)
