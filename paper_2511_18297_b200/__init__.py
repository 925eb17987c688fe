"""B200-native GROOT hot path (arXiv 2511.18297): AIG -> features -> partition ->
edge re-growth -> GraphSAGE forward -> node classes, on sm_100a CUDA kernels
behind the C ABI in include/groot.h. ``api`` mirrors the reference's aigsage
operator API; ``parallel`` shards batch copies / partitions over ranks.
"""
from . import api  # noqa: F401
from ._lib import LIB_PATH, GrootError, GrootInvalidArgument  # noqa: F401
from .api import (  # noqa: F401
    Aig, AugmentedPartition, AugmentedPartitions, CsaCircuit, EdaGraph, Model, PartitionAssignment,
    Prediction, batch, build_plan, classify_aig, core_subgraphs, crossing_fraction, edge_cut, encode,
    footprint_proxy, forward, gen_csa_multiplier, init_model, init_params, load_assignment, load_model,
    materialize, parse_aiger, partition_topo_chunks, predict, predict_full, regrow, save_model, spmm_csr,
    spmm_mean,
)
