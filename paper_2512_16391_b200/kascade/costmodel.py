"""kascade.costmodel (costmodel.py): the analytic cost model; Table 3 presets by default, B200 rows via table="b200"."""
from ..costmodel import (B200_BENCH, FIT_MIN_SEQ, PHASE_DECODE, PHASE_PREFILL, PIPELINE_ANCHORS, PIPELINE_LAYERS,
                         PUBLISHED_BENCH, TABLE_B200, TABLE_PUBLISHED, VALID_MIN_SEQ, BenchRow, CostParams, CostReport,
                         RatioFit, fit_ratios, get_preset, predict_ratios, predict_report, preset_names,
                         report_from_preset, weighted_pipeline_time)

__all__ = ["BenchRow", "CostParams", "CostReport", "get_preset", "predict_ratios", "predict_report", "preset_names",
           "weighted_pipeline_time", "report_from_preset", "fit_ratios", "RatioFit", "PUBLISHED_BENCH", "B200_BENCH",
           "FIT_MIN_SEQ", "VALID_MIN_SEQ", "PHASE_DECODE", "PHASE_PREFILL", "PIPELINE_LAYERS", "PIPELINE_ANCHORS",
           "TABLE_PUBLISHED", "TABLE_B200"]
