"""Synthetic CT phantoms generated on the GPU (reference phantoms.py:1-111).

``generate_phantom(name, dims, spacing)`` returns the same ScalarVolume the
reference builds with numpy -- sphere, shell or torso, air -1000 / tissue 40 /
bone 1200 with 1-2 voxel ramps -- bit for bit: the device kernel evaluates the
same float64 expressions in the same order and rounds with rint.  The device
copy stays resident (attached to the returned volume), so a phantom made for
a render is never uploaded again.
"""

from __future__ import annotations

from .volume import DeviceVolume, ScalarVolume

AIR = -1000
TISSUE = 40
BONE = 1200
SPHERE_PEAK = 1000
SHELL_VALUE = 800
PHANTOM_NAMES = ("sphere", "shell", "torso")


def generate_phantom(name: str, dims=(128, 128, 128), spacing=(1.0, 1.0, 1.0),
                     device: int = 0) -> ScalarVolume:
    """dims is (nx, ny, nz), each >= 8."""
    if name not in PHANTOM_NAMES:
        raise ValueError(f"unknown phantom {name!r}, expected one of {PHANTOM_NAMES}")
    dims = tuple(int(d) for d in dims)
    if any(d < 8 for d in dims):
        raise ValueError(f"phantom dims must be >= 8 per axis, got {dims}")
    dv = DeviceVolume.phantom(name, dims, spacing, device)
    vol = ScalarVolume(dv.download(), tuple(float(s) for s in spacing), dv.value_range)
    vol._attach_device(dv)
    return vol


def device_phantom(name: str, dims, spacing=(1.0, 1.0, 1.0), device: int = 0) -> DeviceVolume:
    """The phantom on the device only (no host copy) -- for benchmarks."""
    return DeviceVolume.phantom(name, dims, spacing, device)
