"""B200-native (sm_100a) RGB-D Gaussian-mixture background model + List-1
colour/depth mask fusion -- the hot path of arXiv 2110.14934's reference
library ``rgbdseg``, rebuilt as hand-written CUDA behind the reference's own
model/segment API.  See DESIGN.md."""
from ._lib import launch_count  # noqa: F401  (fails loudly without the CUDA library)
from .rgbdseg import (  # noqa: F401
    PIXEL_MIXTURE_DTYPE,
    BankMode,
    aos_to_soa,
    soa_to_aos,
    CameraRig,
    DepthRescale,
    FrameMasks,
    FusionState,
    MixtureConfig,
    ModelBank,
    PixelMixture,
    RunConfig,
    SequenceProcessor,
    builtin_scenario_names,
    classify,
    classify_mixtures,
    confusion_counts,
    default_config_json,
    dilate_mask,
    f1_score,
    fuse_step,
    init_mixture,
    init_mixtures,
    match_component,
    match_components,
    register_mask,
    render_scenario,
    reset_state,
    segment_color,
    segment_depth,
    segment_augmented,
    step_mixtures,
    step_pixel,
    update_mixture,
    update_mixtures,
)

from . import dataset, synthetic  # noqa: F401,E402
from .dataset import (  # noqa: F401,E402
    MethodSet,
    SequenceManifest,
    SequenceSource,
    SourceError,
    generate_scenario,
    generate_scenario_from_spec,
    generate_synthetic,
    load_frame,
    load_manifest,
    load_mask_png,
    run_pipeline,
    save_manifest,
    segment_sequence,
)
from .synthetic import ScenarioSpec, builtin_scenario, parse_scenario_spec  # noqa: F401,E402

__all__ = [n for n in dir() if not n.startswith("_")]
