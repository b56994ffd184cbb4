"""CPU-side checks of the C ABI library: it builds, loads, exports every symbol
declared in include/ld.h, and its host-only paths (geometry, argument
validation) behave as documented.  No kernel is launched here."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT, load_golden

HEADER = os.path.join(ROOT, "include", "ld.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(ld_[a-z0-9_]+)\s*\(",
                       text, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def libld():
    from paper_2212_09460_b200 import build, ld
    build.build()
    return ld


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for required in ("ld_sobel_binarize", "ld_hough_accumulate", "ld_hough_peaks",
                     "ld_detect_batch"):
        assert required in names


def test_library_exports_every_declared_symbol(libld):
    out = subprocess.run(["nm", "-D", "--defined-only", libld.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (\w+)$", out, flags=re.M))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    # and the binding wraps all of them under the same names
    assert set(libld.EXPORTS) == set(declared_functions())
    L = ctypes.CDLL(libld.LIB_PATH)
    for n in declared_functions():
        assert hasattr(L, n)


def test_library_is_sm100a_only(libld):
    out = subprocess.run(["cuobjdump", "--list-elf", libld.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_rho_offset_host_geometry(libld):
    for case in load_golden("geometry_pins.json")["rho_offset"]:
        assert libld.ld_rho_offset(case["w"], case["h"]) == case["D"]
    assert libld.ld_rho_offset(0, 5) == -1


def test_status_strings(libld):
    L = libld.lib()
    assert L.ld_status_string(0) == b"LD_OK"
    assert L.ld_status_string(2) == b"LD_ERR_RANGE"


def test_validation_fails_before_any_device_work(libld):
    # NULL gray / bad pitch are rejected on the host, with a detail message
    img = libld.make_image(100, 50, pitch=100)   # pitch not a multiple of 16
    with pytest.raises(libld.LdError) as e:
        libld.ld_sobel_binarize(16, img, 200, None, None, 0, 16, stream=0)
    assert e.value.status == libld.LD_ERR_INVALID_ARG and "pitch" in str(e.value)
    img = libld.make_image(100, 50, pitch=112, row_begin=10, row_end=5)
    with pytest.raises(libld.LdError):
        libld.ld_sobel_binarize(16, img, 200, None, None, 0, 16, stream=0)
    with pytest.raises(libld.LdError) as e:
        libld.ld_hough_peaks(16, 1, 180, 801, 2, 8, 1, 0, 16, 16, 16, 1 << 20, stream=0)
    assert "k 0" in str(e.value)


def test_workspace_sizes_are_consistent(libld):
    img = libld.make_image(1280, 720, 1280, 1280 * 720, 256)
    a = libld.ld_detect_workspace_bytes(img, 180, 4, True)
    b = libld.ld_detect_workspace_bytes(img, 180, 4, False)
    acc = 256 * 180 * (2 * 1469 + 1) * 4
    assert a - b >= acc and a - b < acc + 512
    assert libld.ld_hough_peaks_workspace_bytes(256, 180, 2939, 4) > 0
    assert libld.ld_detect_host_workspace_bytes(img, 180, 4, 32) > 0


def test_validation_of_the_extension_entry_points(libld):
    # every check below happens on the host before any device query
    E = libld.LdError
    with pytest.raises(E) as e:  # hinted voting needs a hint buffer
        libld.ld_hough_accumulate_hint(16, 16, 4, 1, 10, 10, 2, [32768, 0], [0, 32768], 16,
                                       None, 0, stream=0)
    assert e.value.status == libld.LD_ERR_INVALID_ARG
    with pytest.raises(E) as e:  # k = 0
        libld.ld_hough_peaks_hinted(16, 1, 180, 801, 2, 8, 1, 0, 16, 1 << 20, 16, 16, 16, 1 << 20,
                                    stream=0)
    assert e.value.status == libld.LD_ERR_INVALID_ARG
    with pytest.raises(E) as e:  # ratio denominator 0
        libld.ld_hough_peaks_nms(16, 1, 180, 801, 2, 8, 1, 1, 0, 4, 16, 16, 16, 1 << 20, stream=0)
    assert e.value.status == libld.LD_ERR_INVALID_ARG
    with pytest.raises(E) as e:  # NULL peaks
        libld.ld_peak_lines(None, 16, 1, 4, 512, 512, 180, [0] * 180, [0] * 180, 16, 16, stream=0)
    assert e.value.status == libld.LD_ERR_INVALID_ARG
    img = libld.make_image(128, 64, pitch=128)
    with pytest.raises(E) as e:  # max_segments 0
        libld.ld_extract_segments(16, img, 16, 16, 4, 180, [0] * 180, [0] * 180, 20, 40, 0, 16,
                                  16, stream=0)
    assert e.value.status == libld.LD_ERR_INVALID_ARG
    with pytest.raises(E) as e:  # f64 table entry outside [-1, 1] (checked before the device)
        libld.ld_hough_accumulate_f64(16, 16, 4, 1, 10, 10, 2, [2.0, 0.0], [0.0, 1.0], 16,
                                      stream=0)
    assert e.value.status == libld.LD_ERR_RANGE
    with pytest.raises(E) as e:  # f64 mode is limited to 1024 theta bins
        libld.ld_hough_accumulate_f64(16, 16, 4, 1, 10, 10, 1025, [0.0] * 1025, [0.0] * 1025, 16,
                                      stream=0)
    assert e.value.status == libld.LD_ERR_INVALID_ARG


def test_workspace_size_queries_are_host_only(libld):
    assert libld.ld_hough_hint_bytes(256, 1280, 720, 180) >= 64 + 256 * 180 * 8
    assert libld.ld_hough_hint_bytes(0, 1280, 720, 180) == 0
    assert libld.ld_hough_peaks_nms_workspace_bytes(2, 180, 2939) >= 2 * ((180 * 2939 + 31) // 32) * 4
    assert libld.ld_hough_peaks_nms_workspace_bytes(0, 180, 2939) == 0
