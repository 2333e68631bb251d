"""B200-native ADPSGD learner step (arXiv 2110.11199): BLSTM acoustic-model
forward/backward on tcgen05 tensor cores + fused gossip mixing/update, behind a C ABI
(include/adpsgd_b200.h) that mirrors the reference learner/mixing API."""
from .engine import (AsyncMode, DeviceGroup, LearnerGroup, RunRecord, iterations_per_epoch, run_training, write_csv, LrSchedule, LstmObjective, MixKind, ModelDesc, Precision, Strategy,  # noqa: F401
                     StrategyConfig, lr_at, nccl_unique_id, pairing, permutation_for_iteration, strategy_from_name,
                     strategy_name)
from .errors import *  # noqa: F401,F403
