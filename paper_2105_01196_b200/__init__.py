"""B200-native batched bicluster-fitness evaluation (EBIC hot path).

Drop-in for the reference's trend/fitness engine (proj/include/bicseek/trend.hpp):
  * libebic.so      -- sm_100a CUDA kernels behind the C ABI of include/ebic.h
  * csrc/bicseek_trend_device.cpp -- C++ TU replacing proj/src/trend.cpp
  * trend           -- Python mirror of trend.hpp over the C ABI
  * shard           -- multi-GPU row / population sharding (torch.distributed)
  * synth           -- synthetic planted-trend inputs for the benchmark
"""
from .trend import (  # noqa: F401
    EBIC_STORE_AUTO,
    EBIC_STORE_F32,
    EBIC_STORE_F64,
    EbicError,
    Evaluator,
    Population,
    TrendParams,
    device_count,
    evaluate_population,
    fitness,
    read_matrix_tsv,
    row_supports,
    supporting_rows,
)

__version__ = "0.1.0"
