"""B200-native (sm_100a) Mixture-of-Volumetric-Primitives raymarcher.

A drop-in for the reference's forward renderer ``volprim::render``
(/root/reference/proj/src/volprim/march.h:59): per-primitive transforms plus K RGBA voxel
payloads in, image / alpha / per-pixel sample counts out. The compute path is libvpb.so
(hand-written CUDA for sm_100a behind the C-ABI in include/vpb.h); this package is the thin
Python mirror of the reference interface.
"""
from .api import (Camera, Error, ErrorCategory, Frame, MarchConfig, PrimitiveSlab,  # noqa: F401
                  RenderOutput, Renderer, Scene, WindowParams, composite, compose, render,
                  transform_records)

__version__ = "0.1.0"
