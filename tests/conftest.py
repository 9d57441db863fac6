"""Shared fixtures.  GPU tests are marked ``gpu`` and skipped without CUDA;
everything else (oracle vs golden fixtures, host logic, ABI) runs on CPU."""

import dataclasses
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2009_14514_b200 import parse_scene_text  # noqa: E402

TINY_TANK_TEXT = """
domain = 0 0 0  0.4 0.4 0.4
spacing = 0.02
fluid_box = 0.02 0.02 0.02  0.22 0.22 0.22
sound_speed = 30
"""


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and librtssph.so")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def tiny_tank(**overrides):
    scene = parse_scene_text(TINY_TANK_TEXT, name="tiny_tank")
    return dataclasses.replace(scene, **overrides) if overrides else scene


def single_particle_scene(**overrides):
    text = """
    domain = 0 0 0  1 1 2
    spacing = 0.02
    fluid_box = 0.49 0.49 0.99  0.51 0.51 1.01
    sound_speed = 30
    """
    scene = parse_scene_text(text, name="single")
    return dataclasses.replace(scene, **overrides) if overrides else scene


@pytest.fixture
def tank_scene():
    return tiny_tank()
