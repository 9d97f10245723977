"""B200-native Quartet II fully-NVFP4 linear layer.

Drop-in for the hot path of the reference emulator ``nvfp4emu``
(/root/reference/pkg/src/nvfp4emu): same function names and argument
meanings, computed by hand-written sm_100a CUDA in ``libquartet2.so``.
"""

from .rht import CHUNK, SeedPair, derive_stream, hadamard_128, prng_signs, prng_uniform, rht_apply, rht_inverse, sign_mask
from .quantizers import (GROUP, absmax, GUARDED_SCALE_CAP, FP8_RTN_MARGIN, NVFP4Tensor, check_errors, dequantize,
                         deserialize_nvfp4, quantize_rtn, quantize_rtn_46, serialize_nvfp4, set_error_mode)
from .ms_eden import (ErNvfp4Tensor, Pass1Reductions, ms_eden_estimate_pair, ms_eden_quantize, msed, msed_dual, msed_dual_posthoc, msed_stats, set_msed_engine,
                      pass1, pass2,
                      posthoc_quantize)
from .sr import SquareBlockTensor, quantize_square_block, quantize_sr, quantize_sr_46, rht_sr, sr_operand
from .linear_graph import (ABLATIONS, GradPair, LayerConfig, LinearTape, PAIR_DW, PAIR_DX, backward, baseline_config,
                           format_config, forward, gemm, gemm_emulated, parse_config)
from .module import Quartet2Linear, Quartet2LinearFunction, quartet2_linear
from . import formats  # noqa: F401  (formats.py mirror: encode_fp4_rtn, ..., decode_fp8)
from . import ops  # noqa: F401  (torch.ops.quartet2.* custom operators)
from .parallel import ShardedLinearStep, shard_rows, step_seeds

__all__ = [
    "CHUNK", "GROUP", "GUARDED_SCALE_CAP", "FP8_RTN_MARGIN", "SeedPair", "derive_stream", "prng_uniform",
    "sign_mask", "NVFP4Tensor", "quantize_rtn", "quantize_rtn_46", "dequantize", "check_errors",
    "set_error_mode", "ms_eden_quantize", "ms_eden_estimate_pair", "msed", "msed_dual", "msed_dual_posthoc", "msed_stats", "set_msed_engine", "pass1", "pass2", "posthoc_quantize",
    "ErNvfp4Tensor", "Pass1Reductions", "LayerConfig", "LinearTape", "GradPair", "baseline_config", "forward",
    "backward", "gemm", "gemm_emulated", "PAIR_DX", "PAIR_DW", "serialize_nvfp4", "deserialize_nvfp4",
    "quantize_sr", "quantize_sr_46", "absmax", "rht_sr", "sr_operand", "quantize_square_block", "SquareBlockTensor",
    "Quartet2Linear", "Quartet2LinearFunction", "quartet2_linear", "ABLATIONS", "format_config", "parse_config",
    "prng_signs", "rht_apply", "rht_inverse", "hadamard_128", "ShardedLinearStep", "shard_rows", "step_seeds",
]
