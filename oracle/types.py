"""Data-format structs shared with the C-ABI (include/lzb_types.h)."""
from paper_2005_03606_b200._types import *  # noqa: F401,F403
from paper_2005_03606_b200._types import CycleReport, CompressionStats, Field, report_dict  # noqa: F401
