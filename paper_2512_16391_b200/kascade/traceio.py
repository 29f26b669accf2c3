"""kascade.traceio (traceio.py): KSCD v1 traces, plan / report JSON, CSV forms, the synthetic generator."""
from ..host_types import plan_from_dict, plan_to_dict, read_plan, write_plan
from ..kscd_io import (FLAG_XY, MAGIC, coverage_csv, format_report, importance_csv, plans_equal, read_report,
                       read_trace, report_from_dict, report_to_dict, similarity_csv, write_report, write_trace)
from ..kscd_io import VERSION as TRACE_VERSION
from ..synth import SynthConfig, generate_synthetic

DTYPE_F32 = 0                # the header's only dtype code (traceio.py:38)
PLAN_SCHEMA_VERSION = 1      # traceio.py:43
REPORT_SCHEMA_VERSION = 1    # traceio.py:44

__all__ = ["SynthConfig", "generate_synthetic", "read_plan", "read_trace", "write_plan", "write_trace",
           "plan_to_dict", "plan_from_dict", "plans_equal", "report_to_dict", "report_from_dict", "write_report",
           "read_report", "format_report", "similarity_csv", "importance_csv", "coverage_csv", "MAGIC",
           "TRACE_VERSION", "FLAG_XY", "DTYPE_F32", "PLAN_SCHEMA_VERSION", "REPORT_SCHEMA_VERSION"]
