"""Metrics wire format (simulation.py:84-132, report.py:39-72): our
MetricsLog / summarize read the live reference's JSONL and reproduce its
report summary exactly; RunRecorder output follows the same schema."""

import json

from paper_2511_14116_b200.core import Request
from paper_2511_14116_b200.metrics import (MetricsLog, RunRecorder, percentile_nearest_rank,
                                           summarize)

SCHEMA = {  # pkg/README.md:124-141
    "request": {"t", "id", "arrival", "input_len", "output_len", "ttft", "n_tbt", "max_tbt"},
    "iteration": {"t", "duration", "prefill_tokens", "decode_tokens", "batch_requests",
                  "compute_ratio"},
    "interval": {"t0", "t1", "prefill_tokens", "decode_tokens"},
    "failure": {"t", "gpu", "alive"},
    "reconfig_start": {"t", "world", "recovery_latency", "recomputed_tokens", "pcie_bytes"},
    "reconfig_done": {"t", "world"},
    "run_summary": {"t", "completed", "rejected", "preempted", "prefill_tokens", "decode_tokens",
                    "recomputed_tokens", "prefill_throughput", "decode_throughput",
                    "busy_fraction", "compute_ratio_mean", "compute_ratio_max", "unserved"},
}


def test_reference_log_roundtrip_and_summary(golden, tmp_path):
    g = golden("metrics")
    path = tmp_path / "ref.jsonl"
    path.write_text(g["jsonl"])
    log = MetricsLog.read_jsonl(path)
    assert summarize(log) == g["summary"]
    out = tmp_path / "again.jsonl"
    log.write_jsonl(out)
    assert out.read_text() == g["jsonl"]
    for rec in log.records:  # the reference's own records satisfy the schema we emit
        assert SCHEMA.get(rec["kind"], set()) <= set(rec), rec["kind"]


def test_percentile_nearest_rank():
    assert percentile_nearest_rank([5, 1, 3, 2, 4], 50) == 3.0
    assert percentile_nearest_rank([5, 1, 3, 2, 4], 100) == 5.0
    assert percentile_nearest_rank([], 90) == 0.0


def test_recorder_emits_reference_schema(tmp_path):
    from paper_2511_14116_b200.serving import StepBatch
    reqs = [Request(id=i, arrival_time=0.0, input_len=4, output_len=2) for i in range(2)]
    rec = RunRecorder(reqs, world=2)
    # iteration 1: both prompts prefilled (first tokens emitted)
    for r in reqs:
        r.tokens_prefilled, r.tokens_decoded = 4, 1
    rec.iteration(StepBatch(prefill=[(0, 0, 4), (1, 0, 4)]), 0.010, {0: 0.009, 1: 0.010},
                  finished_prefill=[0, 1])
    rec.failure(1, alive=1)
    rec.reconfig(1, 0.075, 3, 1 << 20)
    for r in reqs:
        r.tokens_decoded = 2
    rec.iteration(StepBatch(decode=[(0, 4), (1, 4)]), 0.005, {0: 0.005})
    log = rec.finish()
    kinds = [r["kind"] for r in log.records]
    assert kinds.count("request") == 2 and kinds[-1] == "run_summary"
    for r in log.records:
        assert SCHEMA.get(r["kind"], set()) <= set(r), r["kind"]
    s = summarize(log)
    assert s["requests_completed"] == 2 and s["prefill_tokens"] == 8 and s["decode_tokens"] == 4
    assert abs(s["ttft"]["max"] - 0.010) < 1e-12
    assert abs(s["tbt"]["max"] - 0.080) < 1e-12  # the stall lands in the next token gap
    path = tmp_path / "b200.jsonl"
    log.write_jsonl(path)
    assert json.loads(path.read_text().splitlines()[0])["kind"] == "iteration"
