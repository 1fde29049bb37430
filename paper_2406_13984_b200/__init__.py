"""B200-native GNNDrive (arXiv 2406.13984) sample -> extract hot path.

The product is libfdg.so (CUDA, sm_100a) behind the C ABI in include/fdg.h;
this package is its Python mirror of the reference's interface
(see featdrive.py). Import never falls back to a CPU path.
"""
from .featdrive import (  # noqa: F401
    BufferManager, CudaError, DatasetError, DeviceBuffer, Event, Extractor, Fanouts, FeatdriveError, GraphSAGE, InvalidArgument,
    InvariantViolation, OutOfRange, Pipeline, SampledBatch, Sampler, StandbyTimeout, Stream, Topology, batch_seed,
    device_count, gather, mt_stream, partition_epoch, sample_khop, set_option, trainer_step,
)

__all__ = [
    "BufferManager", "CudaError", "DatasetError", "DeviceBuffer", "Event", "Extractor", "Fanouts", "FeatdriveError", "GraphSAGE",
    "InvalidArgument", "InvariantViolation", "OutOfRange", "Pipeline", "SampledBatch", "Sampler", "StandbyTimeout",
    "Stream", "Topology", "batch_seed", "device_count", "gather", "mt_stream", "partition_epoch",
    "sample_khop", "set_option", "trainer_step",
]
