"""B200-native (sm_100a) PlanarSplatting hot path: differentiable splatting of
rectangular plane primitives into depth / normal / alpha maps with per-plane
gradients, behind the C ABI of include/psplat_b200.h.

Public API mirrors psplat::Renderer (reference proj/core/include/psplat/renderer.hpp).
"""
from .renderer import (  # noqa: F401
    CameraView,
    ForwardResult,
    GradientBuffer,
    LossGrads,
    RenderConfig,
    RenderedMaps,
    Renderer,
    Scene,
    ViewBatch,
    lambda_schedule,
    nccl_unique_id,
)
from .dataio import (Dataset, SceneMeta, load_checkpoint, peek_checkpoint_hash,  # noqa: F401
                     read_map_f32, save_checkpoint, write_dataset, write_map_f32)
from .optimizer import (LossLogRow, OptimConfig, OptimState, Optimizer,  # noqa: F401
                        PlaneInstance, SplatParams)

__version__ = "0.1.0"
