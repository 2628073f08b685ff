"""B200-native Δ-matrix simulated annealing for the QAP (arXiv 1208.2675).

The product is the C-ABI library libqapsa.so (include/qapsa.h, CUDA sm_100a
kernels in csrc/); `qapsa` is its thin ctypes binding and `dist` the
torch.distributed ensemble driver.
"""
from .qapsa import (  # noqa: F401
    QAP_COOL_GEOMETRIC, QAP_COOL_LUNDY_MEES, QapError, Solver, make_schedule, qap_cost,
    qap_create, qap_delta_init, qap_destroy, qap_ensemble_run, qap_get_near_ties, qap_get_state,
    qap_last_kernel_time, qap_reset, qap_sa_run, qap_schedule_bounds, qap_set_option,
    qap_status_str, qap_version,
)

__version__ = "0.1.0"
