"""wavepipe-b200: Hanayo wave-pipeline runtime for B200 (sm_100a).

`schedule` mirrors the reference's schedule API (generate / simulate /
analytics); `runtime` executes an action list on the GPU.  Both sit on the
C ABI of libwavepipe.so (include/wavepipe.h); there is no Python fallback.
"""
from . import schedule  # noqa: F401
from .schedule import *  # noqa: F401,F403
from .runtime import ModelDesc, Runtime, TRANSPORT_IPC, TRANSPORT_LOCAL  # noqa: F401,E402
