"""The request-level entry the reference's CLI and HTTP service share
(service.py:68-94), on the B200 render path.

``prepare_render(volume, payload)`` parses a request body exactly as the
reference does (same error classes and messages) and renders through
``render()``; ``render_request`` returns the PNG bytes and the stats dict the
service sends in the ``X-Render-Stats`` header.  The HTTP server, routing and
volume store of the reference stay out of scope (control plane).
"""

from __future__ import annotations

import json

from .errors import InvalidSettings, IsovalueOutOfRange, UnknownVolume, VoxelrayError
from .imageio import encode_png
from .render import camera_from_dict, render, settings_from_dict
from .transfer import resolve_transfer

STATS_HEADER = "X-Render-Stats"


def status_for(exc: VoxelrayError) -> int:
    """HTTP status of a domain error (service.py:60-65)."""
    if isinstance(exc, UnknownVolume):
        return 404
    if isinstance(exc, (InvalidSettings, IsovalueOutOfRange)):
        return 422
    return 400


def prepare_render(volume, payload: dict):
    """Parse a request body and render; returns the ImageRGBA (service.py:68-88)."""
    if not isinstance(payload, dict) or "camera" not in payload:
        raise InvalidSettings("request body must contain a 'camera' object")
    try:
        camera = camera_from_dict(payload["camera"])
    except (KeyError, TypeError, ValueError) as e:
        raise InvalidSettings(f"camera: {e}") from None
    try:
        tf = resolve_transfer(payload.get("transfer", "grayscale"))
    except (KeyError, TypeError, ValueError) as e:
        raise InvalidSettings(f"transfer: {e}") from None
    try:
        settings = settings_from_dict(payload.get("settings") or {})
    except (TypeError, ValueError) as e:
        raise InvalidSettings(f"settings: {e}") from None
    return render(volume, camera, tf, settings)


def render_request(volume, payload: dict) -> tuple[bytes, dict]:
    """(png bytes, stats dict) for a request body (service.py:91-94)."""
    image = prepare_render(volume, payload)
    return encode_png(image), image.stats.to_dict()


def stats_header(stats: dict) -> dict:
    """The response header carrying the stats (service.py:219-226)."""
    return {STATS_HEADER: json.dumps(stats)}
