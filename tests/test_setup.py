"""Config -> scene resolution (paper_1812_05902_b200.setup) against the reference's
own parse_config_json + build_scene_setup (engine.cpp:228-427), bit for bit."""
import json

import numpy as np
import pytest

from oracle.oracle import Reference, reference_available
from paper_1812_05902_b200 import setup as S

pytestmark = pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")

THIN = [{"type": "aperture", "f_number": 11},
        {"type": "thin_lens", "focal_length_m": 0.105, "diameter_m": 0.03}]


def base(**kw):
    c = {"scene": {"source": {"type": "dots", "extent_m": [0.012, 0.012],
                              "density_per_32px_region": 20, "seed": 7},
                   "medium": {"type": "uniform_gradient_slab", "rho0_kg_m3": 1.225,
                              "grad_kg_m4": [10, 0], "extent_m": [0.048, 0.048], "depth_m": 0.01,
                              "nodes": [25, 25, 5]},
                   "gladstone_dale_m3_kg": 2.26e-4, "ambient_rho_kg_m3": 1.225},
         "geometry": {"z_dot_to_volume_m": 0.25, "z_volume_to_lens_m": 0.73},
         "optics": THIN,
         "sensor": {"resolution": [128, 128], "pitch_m": 1e-5, "bit_depth": 16, "gain": "auto",
                    "distance_m": "auto"},
         "bundle": {"rays_per_source": 1000, "sampling": "stratified", "seed": 1234,
                    "wavelength_m": 5e-7},
         "bos": {"magnification": 0.12}}
    for k, v in kw.items():
        sec, key = k.split("__")
        if sec in ("source", "medium"):
            c["scene"][sec][key] = v
        elif key == "":
            c[sec] = v
        else:
            c[sec][key] = v
    return c


CONFIGS = {
    "bos_uniform": base(),
    # configs/bos_blob.json shape with fewer dots
    "bos_blob": base(source__extent_m=[0.043, 0.043], source__seed=11,
                     medium__type="gaussian_blob_slab", medium__amplitude_kg_m3=0.5,
                     medium__sigma_m=0.004, medium__extent_m=[0.032, 0.032],
                     medium__nodes=[129, 129, 3], sensor__resolution=[560, 560],
                     bundle__rays_per_source=200, bundle__seed=99),
    # configs/demo_aberration.json (magnification measured by the chief-ray probe)
    "aberration": base(source__extent_m=[0.06, 0.06], source__density_per_32px_region=10,
                       source__seed=13, medium__type="none",
                       optics__=[{"type": "aperture", "f_number": 2.8},
                                 {"type": "singlet", "r1_m": 0.103, "r2_m": -0.103,
                                  "thickness_m": 0.005, "glass_index": 1.5, "diameter_m": 0.08}],
                       sensor__resolution=[512, 512], bundle__rays_per_source=300,
                       bundle__seed=6, bos__={}),
    # configs/demo_out_of_focus.json: particles, singlet, explicit z, sensor distance given
    "particles": base(source__={"type": "particles", "count": 50, "diameter_m": 5e-6, "seed": 9,
                                "box_lo_m": [-0.015, -0.015, -0.02], "box_hi_m": [0.015, 0.015, 0.02]},
                      medium__type="none",
                      optics__=[{"type": "aperture", "f_number": 4, "z_m": 0.975},
                                {"type": "singlet", "r1_m": 0.103, "r2_m": 0, "thickness_m": 0.005,
                                 "glass_index": 1.5, "diameter_m": 0.06}],
                      sensor__distance_m=0.2, sensor__resolution=[512, 300],
                      sensor__diffraction_pi_factor=False, bos__={}),
    "fixed_gain_step": base(sensor__gain=1.5e5, trace__={"delta_xi_m": 3e-4, "max_steps": 77},
                            bundle__sampling="uniform-random"),
}


def oracle_calibrate(oracle):
    return lambda scene: oracle.trace(scene, None, with_field=False, accumulate_image=True).image


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_build_scene_matches_reference(oracle, name):
    cfg = CONFIGS[name]
    ref = Reference(json_text=json.dumps(cfg))
    want = ref.scene()
    info_ref = ref.info()
    c = S.parse_config(cfg)
    got, grid, info = S.build_scene(c, calibrate=oracle_calibrate(oracle))
    assert np.array_equal(got.sources, want.sources)
    assert got.pupil_center == want.pupil_center and got.pupil_radius == want.pupil_radius
    assert got.pupil_axis == want.pupil_axis
    assert (got.rays_per_source, got.sampling, got.seed) == \
        (want.rays_per_source, want.sampling, want.seed)
    assert got.delta_xi == want.delta_xi and got.max_steps == want.max_steps
    assert got.d_tau == want.d_tau
    assert bytes(got.sensor) == bytes(want.sensor)
    assert len(got.elements) == len(want.elements)
    for a, b in zip(got.elements, want.elements):
        assert bytes(a) == bytes(b)
    assert info.magnification == info_ref.magnification
    assert info.f_number == info_ref.f_number
    assert info.gain == info_ref.gain
    f_ref = ref.field()
    if f_ref is None:
        assert grid is None
    else:
        f = oracle.field_from_density(grid)
        assert (f.nx, f.ny, f.nz) == (f_ref.nx, f_ref.ny, f_ref.nz)
        assert f.origin == f_ref.origin and f.spacing == f_ref.spacing
        for k in ("n", "gx", "gy", "gz"):
            assert np.array_equal(getattr(f, k), getattr(f_ref, k)), k


def test_gvol_roundtrip_and_recentering(tmp_path, oracle):
    """GVOL1 files load like load_density_volume and are re-centred at Z_D (engine.cpp:31-37)."""
    rng = np.random.default_rng(3)
    g = S.DensityGrid(9, 7, 5, (0.1, 0.2, 0.3), (0.003, 0.003, 0.0025),
                      (1.225 + 0.01 * rng.random(9 * 7 * 5)).astype(np.float32))
    p = str(tmp_path / "v.gvol")
    S.save_gvol(g, p)
    cfg = base(medium__={"type": "gvol", "path": p}, bundle__rays_per_source=100,
               sensor__gain=1e5)
    ref = Reference(json_text=json.dumps(cfg))
    got, grid, info = S.build_scene(S.parse_config(cfg))
    f_ref = ref.field()
    f = oracle.field_from_density(grid)
    assert f.origin == f_ref.origin
    assert np.array_equal(f.n, f_ref.n) and np.array_equal(f.gz, f_ref.gz)
    assert got.delta_xi == ref.scene().delta_xi and got.max_steps == ref.scene().max_steps


def test_config_errors_match_reference_messages():
    with pytest.raises(S.ConfigError, match="optics chain must not be empty"):
        S.parse_config({"optics": []})
    with pytest.raises(S.ConfigError, match="unknown medium type"):
        S.parse_config(base(medium__type="fog"))
    with pytest.raises(S.ConfigError, match="rays_per_source must be >= 1"):
        S.parse_config(base(bundle__rays_per_source=0))


def test_quantize_matches_reference():
    rng = np.random.default_rng(5)
    img = rng.random((64, 64)) * 1e-3
    img[0, :8] = [0.0, 1e9, 0.5 / 7e4, 1.5 / 7e4, 2.5 / 7e4, -1.0, np.nextafter(0.5, 0) / 7e4, 3e-5]
    gain = 7e4
    assert np.array_equal(S.quantize(img, 16, gain), Reference.quantize(img, 16, gain))
    assert np.array_equal(S.quantize(img, 10, gain), Reference.quantize(img, 10, gain))
