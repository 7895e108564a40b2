"""CPU-only checks (no GPU needed): the glibc libm replicas used by the
kernels against this host's libm, the C-ABI library's exported symbols, the
config mirror against the reference's defaults/validation, and the
reference oracle's own known answers (test_output.txt)."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from paper_2203_02300_b200.config import FIELDS, Config, ConfigError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dco_gpu.h")
LIB = os.path.join(ROOT, "paper_2203_02300_b200", "libdco_gpu.so")


@pytest.fixture(scope="module")
def libm_check(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("libm") / "libm_check")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe, os.path.join(ROOT, "oracle", "libm_check.c"), "-lm"],
                   check=True)
    return exe


@pytest.mark.parametrize("mode,n", [("exp_rand", 2000000), ("hypotf", 2000000), ("hypot", 2000000),
                                    ("atan2f", 2000000)])
def test_libm_replica_random(libm_check, mode, n):
    r = subprocess.run([libm_check, mode, str(n)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.split()[2] == "0"


@pytest.mark.parametrize("lam", [10.0, 3.5])
def test_libm_replica_exp_ad_domain(libm_check, lam):
    """Every float |dI| in [0,1] (stride 7 here; stride 1 in the slow test) for
    the AD term argument -(double)f*255/lambda_ad (stereo.cpp:142)."""
    r = subprocess.run([libm_check, "exp_ad", str(lam), "7"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.slow
def test_libm_replica_exp_ad_exhaustive(libm_check):
    r = subprocess.run([libm_check, "exp_ad", "10", "1"], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.split()[1] == "1065353217", r.stdout + r.stderr


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|uint64_t|size_t|const char\*)\s+(dco_\w+)\(", src, re.M)))


def test_cabi_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        from paper_2203_02300_b200 import build

        build.build(verbose=False)
    names = declared_functions()
    assert len(names) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (dco_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    # the library loads without a GPU and reports its ABI version
    lib = ctypes.CDLL(LIB)
    assert lib.dco_abi_version() == 3
    from paper_2203_02300_b200 import native

    assert set(native.SIGNATURES) == set(names)


def test_cabi_without_gpu_fails_loudly():
    lib = ctypes.CDLL(LIB)
    h = ctypes.c_void_p()
    st = lib.dco_create(0, ctypes.byref(h))
    import torch

    if not torch.cuda.is_available():
        assert st == 4  # DCO_CUDA: no CPU fallback


def test_config_mirror_matches_reference(ref):
    c = ref.default_config()
    mine = Config()
    for n, _, _ in FIELDS:
        assert getattr(c, n) == getattr(mine, n), n
    lib = ctypes.CDLL(LIB)
    g = Config(d_max=1)
    lib.dco_config_default(ctypes.byref(g))
    for n, _, _ in FIELDS:
        assert getattr(g, n) == getattr(mine, n), n


BAD = [dict(d_min=5, d_max=5), dict(t_low=0.07), dict(t_depth=1.5), dict(lambda_s=0.0), dict(gamma_l=-1.0),
       dict(census_window_w=8), dict(census_window_w=11), dict(cross_arm_l2=18), dict(cross_color_tau=0.0),
       dict(box_radius=0), dict(gauss_sigma=0.0), dict(confidence_offset_k=0.0), dict(hist_iterations=-1),
       dict(focal_px=0.0), dict(solver_max_iter=0), dict(d_min=-1, d_max=4)]


@pytest.mark.parametrize("bad", BAD, ids=lambda b: ",".join(b))
def test_config_validation_matches_reference(ref, bad):
    lib = ctypes.CDLL(LIB)
    c = Config(**bad)
    with pytest.raises(ConfigError):
        ref.validate(c)
    msg = ctypes.create_string_buffer(256)
    lib.dco_config_validate.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]
    assert lib.dco_config_validate(ctypes.byref(c), msg, 256) == 5
    with pytest.raises(ConfigError) as e:
        ref.validate(c)
    assert msg.value.decode() == str(e.value)


def test_reference_stereo_kat(ref):
    """criterion_stereo_oracle: ratio=0.993448 valid=74781 (test_output.txt:28)."""
    cfg = Config()
    f = ref.render_synth_frame(960, 320, 0, square_size=160, square_x0=400.0, square_y0=80.0, shift_x=0.0, seed=7)
    lq, rq = ref.downsample_half(f["left"]), ref.downsample_half(f["right"])
    arms = ref.build_cross_windows(lq, cfg)
    d = ref.refine_disparity_histogram(
        ref.select_disparity_wta(ref.aggregate_costs(ref.compute_cost_volume(lq, rq, arms, cfg), arms)), arms, 2)
    sp = ref.disparity_to_sparse_depth(d, cfg, 960, 320)
    valid = np.isfinite(sp)
    dq = cfg.focal_px * cfg.baseline_m / sp[valid].astype(np.float64) / 2.0
    truth = np.where(f["gt_depth"][valid] == 1.0, 24.0, 12.0)
    assert valid.sum() == 74781
    assert "%.6f" % ((np.abs(dq - truth) <= 1.0).sum() / valid.sum()) == "0.993448"


def test_reference_alpha_kat(ref):
    # acceptance.cpp:163-170: alpha(0) = 1 - exp(-1.25), printed 0.713495
    a = ref.adaptive_alpha(0, Config())
    assert abs(a - (1.0 - np.exp(-1.25))) < 1e-9 and "%.6f" % a == "0.713495"


def test_golden_mask_fixture_present():
    from oracle.pgm import read_pgm

    m = read_pgm(os.path.join(ROOT, "tests", "golden", "golden_mask.pgm"))
    assert m.shape == (96, 160) and set(np.unique(m)) <= {0, 255} and (m > 0).sum() > 100
