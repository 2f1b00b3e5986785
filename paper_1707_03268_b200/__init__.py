"""B200-native DPM score path (arXiv 1707.03268): drop-in for cpdetect's scoring.

Reference-compatible entry points (``cpdetect.correlation`` /
``cpdetect.detection``, pruning off) run on hand-written sm_100a kernels in
``lib/libdpm_b200.so`` (C ABI: ``include/dpm_b200.h``):

  K1 project    - HOG level -> rank-R basis          (HBM-bound)
  K2 correlate  - shortened multi-filter correlation (FP32 FFMA implicit GEMM)
  K3 place      - penalised window max / GDT + argmax (FP64, bit-exact)
  K4 assemble   - root + shifted parts + bias, tau compaction

``PyramidScorer`` batches whole pyramids of many images through one launch
per kernel; ``features`` builds the 32-channel HOG pyramids of raw images
on the device.  There is no CPU fallback.
"""

from .correlation import (ScoreMap, correlate3_cp, correlate3_full, cp_multiplications,
                          cp_partial_stack, full_multiplications, theoretical_gain,
                          valid_support)
from .detection import (_placement_grid, best_part_placement, calibrate_thresholds,
                        cp_score_hypothesis, deformation_penalty, dense_detect, detect,
                        score_hypothesis, validate)
from . import formats  # noqa: F401
from .evaluation import RocPoint, match_detections, nms, nms_records, roc_eval
from .errors import CpdetectError, DeviceError, FormatError, NumericError, ValidationError
from .features import HogBuilder, extract_hog_pyramid
from .pipeline import PyramidScorer, cores_from_stacked, detect_batch, score_pyramid
from .plancache import clear_plan_cache, plan_cache_info
from .types import (CPModel, DecomposedModel, DecomposedPart, Detection, DetectStats,
                    Hypothesis, PartModel, PartSpec)

__version__ = "0.1.0"

__all__ = [
    "CPModel", "CpdetectError", "DecomposedModel", "DecomposedPart", "Detection",
    "DetectStats", "DeviceError", "FormatError", "Hypothesis", "NumericError", "PartModel",
    "PartSpec", "PyramidScorer", "ScoreMap", "ValidationError", "_placement_grid",
    "best_part_placement", "cores_from_stacked", "correlate3_cp", "correlate3_full",
    "cp_multiplications", "cp_partial_stack", "cp_score_hypothesis", "deformation_penalty",
    "dense_detect", "detect",
    "calibrate_thresholds", "score_pyramid", "detect_batch", "nms", "nms_records", "match_detections", "roc_eval",
    "RocPoint", "full_multiplications", "score_hypothesis", "theoretical_gain",
    "HogBuilder", "extract_hog_pyramid", "clear_plan_cache", "plan_cache_info",
    "valid_support", "validate",
]
