"""Viewer frames (session.py:381-405, protocol.py:29-55): the selection overlay
and RGBA8 quantisation.  `View.render_rgba` does both on the device in the
raster's epilogue (rcgs_render_rgba); these host helpers restate the reference's
own functions for callers holding host images."""

from __future__ import annotations

import struct

import numpy as np

from .errors import ValidationError

HIGHLIGHT_COLOR = (1.0, 0.8, 0.1)   # session.py:52
HIGHLIGHT_STRENGTH = 0.45           # session.py:53
FRAME_MAGIC = b"RCGS"
FORMAT_RAW = 0
HEADER = struct.Struct("<4sIIII")


def overlay(image: np.ndarray, bits: np.ndarray, color=HIGHLIGHT_COLOR,
            strength: float = HIGHLIGHT_STRENGTH) -> np.ndarray:
    """image[bits] = (1 - s) image[bits] + s color (session.py:398-401)."""
    image = np.array(image, dtype=np.float64, copy=True)
    if bits is not None and bits.any():
        image[bits] = (1.0 - strength) * image[bits] + strength * np.asarray(color)
    return image


def image_to_rgba(image: np.ndarray) -> np.ndarray:
    """Float (H, W, 3) image -> uint8 RGBA, alpha 255 (protocol.py:29-38)."""
    image = np.asarray(image, dtype=np.float64)
    if image.ndim != 3 or image.shape[2] != 3:
        raise ValidationError(f"expected (H, W, 3) image, got {image.shape}")
    rgba = np.empty(image.shape[:2] + (4,), dtype=np.uint8)
    rgba[..., :3] = np.rint(np.clip(image, 0.0, 1.0) * 255.0).astype(np.uint8)
    rgba[..., 3] = 255
    return rgba


def encode_frame(rgba: np.ndarray) -> bytes:
    """Header-prefixed raw frame (protocol.py:41-55, "raw" format)."""
    rgba = np.ascontiguousarray(rgba, dtype=np.uint8)
    if rgba.ndim != 3 or rgba.shape[2] != 4:
        raise ValidationError(f"expected (H, W, 4) RGBA, got {rgba.shape}")
    height, width = rgba.shape[:2]
    payload = rgba.tobytes()
    return HEADER.pack(FRAME_MAGIC, width, height, FORMAT_RAW, len(payload)) + payload
