"""B200-native VATE hot path: a drop-in for slidecard's ingest / advance / estimate.

Same public names as the reference package's path (slidecard/__init__.py:10-50,
the hot-path subset): the AT pool, the estimator functions and the slice
pipeline, backed by hand-written sm_100a CUDA kernels in libvate_b200.so.
Importing this package fails loudly if the library has not been built.
"""

from .errors import ConfigError, TraceError, TraceOrderError, TraceParseError
from .pools import (LOW_DEVIATION, PARTITIONS, TAIL_REMAINDER, AtPool, DrPool, MaintenanceReport,
                    TsPool, make_pool)
from .estimator import (EstimateReport, EstimatorConfig, HostReports, estimate_host,
                        estimate_hosts, estimate_hosts_soa, estimate_linear, host_cells,
                        inactive_virtual_counts, pair_cells, record_packed, record_pairs,
                        reports_from_counts, reports_from_counts_soa)
from .pipeline import Pipeline, SliceStats, SlidingHostSet
from .counters import MAX_K, TS_UNSET, WindowConfig, ats_bits, dr_bits

__version__ = "0.1.0"

__all__ = [
    "AtPool", "ConfigError", "DrPool", "TsPool", "TS_UNSET", "dr_bits", "EstimateReport", "EstimatorConfig", "HostReports",
    "LOW_DEVIATION", "MAX_K", "MaintenanceReport", "PARTITIONS", "Pipeline", "SliceStats",
    "SlidingHostSet", "TAIL_REMAINDER", "TraceError", "TraceOrderError", "TraceParseError",
    "WindowConfig", "ats_bits", "estimate_host", "estimate_hosts", "estimate_hosts_soa",
    "estimate_linear", "host_cells", "inactive_virtual_counts", "make_pool", "pair_cells",
    "record_packed", "record_pairs", "reports_from_counts", "reports_from_counts_soa",
]
