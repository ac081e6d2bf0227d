"""B200-native P-HGRMS (arXiv 1306.5390) denoise path.

The C++ reference API (include/phgrms/denoise.hpp) re-served from sm_100a
kernels through the C ABI in include/phgrms_b200.h.  See DESIGN.md.
"""
from ._lib import LIB_PATH, CudaError, InvalidArgument, lib  # noqa: F401
from .phgrms import (  # noqa: F401
    BorderMode,
    CardinalityMap,
    DenoiseParams,
    DenoiseResult,
    EngineMode,
    EngineSpec,
    PsnrValue,
    GrayImage,
    NoiseSpec,
    PassStats,
    RowBlock,
    SynthKind,
    cardmap,
    compute_cardinality,
    denoise,
    denoise_batch,
    denoise_sharded,
    denoise_pass,
    denoise_pgm_file,
    inject_sp_noise,
    format_db,
    kernel_name,
    mse,
    psnr,
    parallel_for_rows,
    residual_noise_count,
    rms_replacement,
    row_blocks,
    similar,
    synth_image,
    write_p2,
)
