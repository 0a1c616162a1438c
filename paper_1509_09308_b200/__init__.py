"""B200-native (sm_100a) Winograd fast convolution, F(2x2,3x3) and F(4x4,3x3).

Drop-in for the hot path of the reference ``winoconv`` package
(``winograd_forward`` and the ``f2x2``/``f4x4``/``*-fx`` algorithm names),
computed by hand-written CUDA kernels in ``libwino.so`` (C ABI:
``include/wino.h``).  Importing this package loads the CUDA library and
fails loudly if it is missing: there is no CPU fallback.
"""
from ._lib import version  # noqa: F401  (loads libwino.so or raises)
from .commands import (ACCURACY_ALGOS, BENCH_ALGOS, cmd_accuracy, cmd_bench, layer_inputs,
                       parse_algo, run_layer)
from .direct import direct_forward
from .engine import (FilterCache, TileGrid, WinogradPlan, get_plan, multiply_stage_flops,
                     shared_filter_cache, tile_count, winograd_forward, winograd_grad_inputs,
                     winograd_grad_weights, grad_weights_device)
from .layer import LayerConfig, OpCounter, WinogradAlgorithm, builtin, builtin_sizes, gflops_direct
from .suites import LayerSuite, get_suite, vgg_e, vgg_e_accuracy
from .tensors import Precision, Tensor4, fill_uniform, max_abs_error, quantize_fp16

__version__ = "0.2.0"

__all__ = [
    "Precision", "Tensor4", "fill_uniform", "quantize_fp16", "max_abs_error",
    "LayerConfig", "gflops_direct", "WinogradAlgorithm", "builtin", "builtin_sizes",
    "OpCounter", "FilterCache", "TileGrid", "tile_count", "multiply_stage_flops",
    "winograd_forward", "winograd_grad_inputs", "winograd_grad_weights", "grad_weights_device", "shared_filter_cache", "WinogradPlan",
    "get_plan", "run_layer", "cmd_bench", "cmd_accuracy", "layer_inputs", "parse_algo",
    "BENCH_ALGOS", "ACCURACY_ALGOS", "direct_forward",
    "LayerSuite", "get_suite", "vgg_e", "vgg_e_accuracy", "version", "__version__",
]
