"""B200-native population-vectorized off-policy update path (TD3 / SAC + replay + PBT).

The compute lives in libpbrl_b200.so (hand-written sm_100a CUDA behind the C ABI in
include/pbrl_b200.h); this package is the host mirror of the reference pbrl API.
"""
from .errors import (ConfigError, CudaError, DataStarvationError, DegeneratePopulationError,
                     NcclError, NotReadyError, PbrlError, ResourceError, ShapeError, UsageError)
from .pbrl import (NETS, PBTState, RngSequence, RngStream, SacHyper, SacPrior, SacState, Td3Hyper,
                   Td3Prior, Td3State, Transition, TransitionBatch, DeviceReplay, EvolvePlan,
                   HyperRange, make_sac_state, make_synthetic_batches, make_td3_state, mix64,
                   pbt_apply_returns_reset, pbt_evolve_trainer, pbt_plan, pbt_rank,
                   sac_update_step, sample_batch, td3_update_step, update_k_steps, act, sac_act,
                   save_checkpoint, load_checkpoint, serialize_state, deserialize_state,
                   update_k_from_replay, slice_member, set_member,
                   SnapshotMailbox, actor_refresh, LambdaSchedule, DvDConfig, DvdHook,
                   DvdLossOut, dvd_lambda, dvd_policy_hook, dvd_embed, dvd_loss,
                   median_pairwise_distance, CEMState, cem_init, cem_resample, cem_update)

__all__ = [n for n in dir() if not n.startswith("_")]
