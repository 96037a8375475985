"""B200-native ReLibra MoE-layer hot path.

Drop-in for the planner API of the reference package ``moebalance`` (re-exported names of
pkg/src/moebalance/__init__.py:3-66 that lie on the MoE-layer path), backed by
``libmb_planner.so`` (C++ planners) and ``libmb_sm100.so`` (sm_100a data-plane kernels):

    from paper_2605_08639_b200 import build_topology, HardwareProfile, anneal_reorder, ...

The data plane (replayed-routing histogram, permute/dispatch, tcgen05 grouped-GEMM expert
FFN, combine, replica push / gradient reduce) lives in ``moe_layer`` / ``kernels``.
"""

from .cluster import (ClusterTopology, HardwareProfile, TrafficClass, b200_box_topology, b200_profile,
                      build_topology, classify_traffic, relay_gpu)
from .loads import (CostEstimate, LoadVector, SmoothingConfig, comm_row_times, comm_time, comp_time,
                    compute_loads, flow_matrix, lse, moe_time, smoothed_moe_time)
from .policies import (POLICIES, PlanBundle, SimConfigs, SimReport, build_policy_bundle, compare_report,
                       evaluate_bundle, run_baseline, solve_tasks)
from .reordering import (AnnealConfig, ReorderPlan, SamplePlacement, anneal_reorder, anneal_reorder_device,
                         anneal_reorder_layers_device,
                         anneal_sample_placement,
                         apply_plan, greedy_sample_initial, lpt_initial, rewrite_trace_matrices, static_plan)
from .replication import (InstanceTooLargeError, ReplicaConfig, ReplicaPlacement, ReplicationEntry,
                          ReplicationPlan, SplitPlan, candidate_gpus, greedy_replicate, replica_memory, round_split,
                          solve_token_split_lp, validate_placement, validate_split)
from .traces import (ModelProfile, RoutingTrace, SampleTable, TraceFormatError, ZipfRouting, aggregate_batch,
                     build_trace, hot_expert_intersection, load_trace, realize_tokens, save_trace, skewness,
                     top_k_experts)
from .planio import (PlanFormatError, chain_seeds, load_plan_bundle, load_reorder_plan, load_replication_plan,
                     replication_plan_from_dict, replication_plan_to_dict, save_reorder_plan, save_replication_plan,
                     solve)
from ._native import LPError, NativeLibraryError

__version__ = "0.1.0"
