"""Strategy names shared with the reference's configuration surface.

The analytic comparison systems of `/root/reference/pkg/src/chunkstar/baselines.py`
(static offload, DDP, L2L closed forms and the max-scale ladder walk) are
OUT OF SCOPE for this build ("analytic comparison systems, not
the step").  Only the names the hot-path configuration and the reference's
acceptance-test imports need are defined; the functions raise.
"""

from enum import Enum

STATIC_OFFLOAD = "static_offload"
DDP = "ddp"
L2L = "l2l"
CHUNK = "chunk"


class FailureReason(str, Enum):
    NONE = "none"
    GPU_OOM = "gpu_oom"
    CPU_OOM = "cpu_oom"


def _out_of_scope(name: str):
    def fn(*args, **kwargs):
        raise NotImplementedError(
            "%s is an analytic comparison baseline of the reference simulator; "
            "it is out of scope for the B200 chunk-step build (see DESIGN.md)" % name)
    fn.__name__ = name
    return fn


simulate_static_offload = _out_of_scope("simulate_static_offload")
simulate_ddp = _out_of_scope("simulate_ddp")
simulate_l2l = _out_of_scope("simulate_l2l")
max_feasible_scale = _out_of_scope("max_feasible_scale")
