"""B200-native (sm_100a) training hot path of arXiv 2109.07893: a
snapshot-sequence dynamic GNN (GCN per snapshot + LSTM / M-product per
vertex timeline) with graph-difference snapshot transfer, snapshot-partitioned
multi-GPU execution and gradient checkpointing over time blocks.

Drop-in for the reference `dtgnn` model/trainer API on that path; the
compute runs in hand-written CUDA kernels (`libdgnn_b200.so`, C ABI in
`include/dgnn_b200.h`).  There is no CPU execution path: calling the
engines without a CUDA device or without the built library raises.
"""

__version__ = "0.1.0"

from .errors import (ConfigError, CorruptDeltaError, DeviceError, DtgnnError, EdgeListParseError,  # noqa: F401
                     InputError, ProtocolError)
from .graph import (DynamicGraph, FeatureSequence, MMatrix, SparseMatrix, build_m_matrix,  # noqa: F401
                    degree_features, m_transform_features, m_transform_graph)
from .labels import LabelSet, sample_link_prediction_sets  # noqa: F401
from .params import ModelConfig, init_params, parameter_count  # noqa: F401
from .api import (ActivationLedger, AdamState, BlockPlan, CommLedger, SnapshotPartition, TrainingData,  # noqa: F401
                  TransferLedger, backward_checkpoint, backward_full, distributed_epoch,
                  adam_step, init_adam, plan_snapshot_partition, prepare_training_data,
                  model_forward_frames, train_distributed, train_epochs)
from .wire import read_delta_stream, train_report, write_delta_stream  # noqa: F401
from .ops import (SnapshotDelta, apply, diff, lstm_block_backward, lstm_block_forward,  # noqa: F401
                  naive_cost, normalize_laplacian, spmm, spmm_transpose, stream_block)
