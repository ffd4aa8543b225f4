"""B200-native volume ray casting: the voxelray render path on sm_100a.

Drop-in for the reference package's render path (voxelray.render.render and
its block prep, /root/reference/pkg/src/voxelray): same classes, functions,
arguments, errors and outputs; the per-voxel and per-ray work runs in the
hand-written CUDA kernels of csrc/ behind the C ABI in include/voxelray_b200.h.
"""

from .blocks import Block, BlockGrid, block_stats, cull_empty, decompose, traversal_order, with_visibility
from .errors import (
    DeviceError,
    DimensionMismatch,
    DuplicatePosition,
    EmptyBlock,
    InconsistentGeometry,
    InvalidBlockSpec,
    InvalidSettings,
    IsovalueOutOfRange,
    NonUniformSpacing,
    SizeMismatch,
    UnknownVolume,
    VoxelrayError,
)
from .ingest import DeviceVolumeCache, assemble_volume_device, ingest_raw, volume_id
from .measure import ball_counts, ball_measure, threshold_count, threshold_measure, threshold_volume_mm3
from .phantoms import PHANTOM_NAMES, device_phantom, generate_phantom
from .quality import convergence_study, psnr, ssim
from .render import (
    Camera,
    ImageRGBA,
    OrthographicCamera,
    Renderer,
    RenderSettings,
    RenderStats,
    camera_from_dict,
    composite_step,
    generate_ray,
    render,
    render_views,
    settings_from_dict,
    shade_headlight,
)
from .sampling import gradient, sample, sample_tricubic, sample_trilinear
from .transfer import (
    ClassifiedLUT,
    PreintegratedTable,
    TransferFunction,
    build_lut,
    build_preintegrated,
    get_preset,
    preclassify_volume,
    resolve_transfer,
    transfer_from_dict,
    transfer_from_points,
    windowed_transfer,
)
from .volume import DeviceVolume, ScalarVolume, load_raw, make_volume

__version__ = "0.1.0"
