"""paper_2404_16221_b200 — B200-native NeRF-XL distributed ray-march / composite path.

Drop-in for the reference ``volray`` package's hot path (distsim._run_ray and its
callees).  The API names mirror reference ``volray/__init__.py``; the work runs in
hand-written sm_100a kernels behind the C ABI in ``include/vr_capi.h``.
"""
from . import _lib
from .comm import all_gather_packets, gather_packets, owned_regions
from .engine import (
    PROTOCOLS,
    RayAggregate,
    SampleBatch,
    VolumePool,
    canonical_protocol,
    render_image,
    render_ray,
    spawn,
    write_ppm,
)
from .errors import (
    CapacityError,
    DegenerateSplitError,
    GradientOverflowError,
    InsufficientPointsError,
    NegativeLossError,
    NoPointsError,
    NonFiniteInputError,
    OutOfBoundsError,
    ParamNotOwnedError,
    ProtocolMismatchError,
    VrError,
)
from .fields import (
    AnalyticRegion,
    ConstantBox,
    GaussianBlob,
    GaussianBlobs,
    HashGridConfig,
    HashGridMLP,
    RegionField,
    Scene,
    SumField,
    VoxelGrid,
    VoxelRegion,
    field_from_json,
    scene_from_json,
)
from .geometry import Aabb, Camera, Ray, camera_ray_dirs, camera_rays, rays_to_soa, soa_rays, unit, vec3
from .partition import (
    LeafNode,
    PartitionTree,
    PointCloud,
    SplitNode,
    balance_report,
    build_tree,
    choose_split,
    default_root_box,
    grid_tree,
    rays_to_points,
    load_tree,
    locate,
    locate_many,
    save_tree,
    tree_from_json,
    tree_to_json,
)
from .segments import (
    DeviceFieldView,
    DistributedLossProbe,
    Field,
    ParamRef,
    SampleInterval,
    SegmentAggregate,
    aggregate_segment,
    aggregate_segments,
    compose_distortion,
    compose_packets,
    compose_render,
    fill_samples,
    identity_aggregate,
    local_gradient_fd,
)
from .stats import CommStats, stats_json

__version__ = "0.1.0"
