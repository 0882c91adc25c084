"""Golden vectors for the native trace reader (ks_trace_parse), made by
running the REFERENCE parser (kernsim.trace.parse_trace, trace.py:281-328)
on crafted edge-case documents.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_parse_golden.py

Writes tests/golden/parse_golden.json.gz: per case the document text and
either the reference's error (class name, and the two ids of an
OverlapViolation) or document_to_object() of the parsed document.  Cases on
which the reference raises a non-KernsimError (e.g. decimal.InvalidOperation
for NaN times) are recorded with error "<non-kernsim:Type>".
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from kernsim.errors import KernsimError, OverlapViolation  # noqa: E402
from kernsim.trace import document_to_object, parse_trace  # noqa: E402

OUT = Path(__file__).resolve().parent / "parse_golden.json.gz"
HEAD = '"schema_version": 1, "time_unit": "microseconds"'


def doc(events="", markers=None, extra=""):
    parts = [HEAD, f'"events": [{events}]']
    if markers is not None:
        parts.append(f'"layer_markers": [{markers}]')
    if extra:
        parts.append(extra)
    return "{" + ", ".join(parts) + "}"


def ev(i, kind="CpuOther", lane="cpu:0", start=0, dur=1, name='"x"', extra=""):
    s = f'{{"id": {i}, "kind": "{kind}", "name": {name}, "lane": "{lane}", "start": {start}, "duration": {dur}'
    return s + (", " + extra if extra else "") + "}"


def cases():
    c = {}
    # -- time conversion: literals, shortest repr, strings
    times = ["0", "1", "0.1", "0.30000000000000004", "1.2345678", "12.345", "0.0005", "0.0015",
             "2.4995", "2.4994", "1e-7", "2.5e3", "1E2", "123456.7891234567891",
             "9007199254.740993", "1234567.8915", "-0.0", "0.00049999999999999999",
             "0.000499999999999999", "7.00050000000000000001", "1e-400", "123456789012.3456789",
             '"12.5"', '" 7.0005 "', '"1_000"', '"+.5e-1"', '"1."', '".5"', '"1__0.5"',
             '"-0.0004"', "-0.0004", "9223372036854", "4.9999999999999996e-4"]
    for k, t in enumerate(times):
        c[f"time_{k}"] = doc(ev(0, start=t, dur=t))
    for k, t in enumerate(['"abc"', "true", "null", "[1]", "{}", '"1e"', "-1", "-0.0005",
                           '"0x10"', '""']):
        c[f"badtime_{k}"] = doc(ev(0, start=t))
    c["nan_time"] = doc(ev(0, start="NaN"))
    c["inf_time"] = doc(ev(0, dur="Infinity"))
    # -- ids / ints
    c["id_true"] = doc(ev("true"))
    c["id_false"] = doc(ev("false"))
    for k, v in enumerate(["-1", "1.5", '"3"', "null", "1e2", "-0"]):
        c[f"bad_id_{k}"] = doc(ev(v))
    c["missing_id"] = doc('{"kind": "CpuOther", "name": "x", "lane": "cpu:0", "start": 0, "duration": 1}')
    for k, v in enumerate(["-1", "1.0", '"5"', "true", "null"]):
        c[f"corr_{k}"] = doc(ev(0, extra=f'"correlation": {v}'))
        c[f"size_{k}"] = doc(ev(0, extra=f'"size_bytes": {v}'))
    # -- names and strings
    for k, nm in enumerate(['"k\\u00e9\\u00e9"', '"\\"q\\"\\\\"', '"\\ud83d\\ude00"', "42", "true",
                            "null", "-0", '"\\ud800x"', '"memcpy_dtoh_async"', '"memcpy_dto"',
                            '"tab\\tnew\\nline\\/"', '"é中"']):
        c[f"name_{k}"] = doc(ev(0, name=nm))
    c["name_missing"] = doc('{"id": 0, "kind": "CpuOther", "lane": "cpu:0", "start": 0, "duration": 1}')
    c["lane_escaped"] = doc(ev(0, lane="cpu\\u003a0"))
    c["key_escaped"] = doc('{"\\u0069d": 3, "kind": "CpuOther", "name": "x", "lane": "cpu:0", "start": 0, "duration": 1}')
    c["dup_keys"] = doc('{"id": 0, "kind": "CpuOther", "name": "x", "lane": "cpu:0", "start": 5, "start": 7, "duration": 1}')
    c["unknown_nested"] = doc(ev(0, extra='"vendor": {"a": [1, 2, {"b": null}], "c": "}]"}'), extra='"extra": [true]')
    for k, ln in enumerate(["xpu:0", "cpu:", "cpu", ":0", "gpu:0:1"]):
        c[f"lane_{k}"] = doc(ev(0, lane=ln))
    c["lane_int"] = doc('{"id": 0, "kind": "CpuOther", "name": "x", "lane": 5, "start": 0, "duration": 1}')
    # -- kinds / lane classes / sync
    c["kind_bad"] = doc('{"kind": "Nope"}')
    c["kind_null"] = doc(ev(0, kind="CpuOther").replace('"CpuOther"', "null"))
    c["kind_missing"] = doc('{"id": 0}')
    c["gpu_no_corr"] = doc(ev(0, kind="GpuKernel", lane="gpu:0:1"))
    c["gpu_on_cpu"] = doc(ev(0, kind="GpuKernel", lane="cpu:0", extra='"correlation": 1'))
    c["cpu_on_gpu"] = doc(ev(0, kind="CpuApi", lane="gpu:0:1"))
    c["comm_on_cpu"] = doc(ev(0, kind="Comm", lane="cpu:0"))
    c["comm_ok"] = doc(ev(0, kind="Comm", lane="comm:ring0"))
    c["sync_target_non_sync"] = doc(ev(0, extra='"sync_target": "gpu:0:1"'))
    c["sync_target_bad"] = doc(ev(0, kind="Sync", extra='"sync_target": "gpux"'))
    c["sync_ok"] = doc(", ".join([ev(0, kind="Sync", extra='"sync_target": "gpu:0:9"'),
                                  ev(1, kind="Sync", start=5), ev(2, kind="DataLoad", start=10)]))
    # -- document level
    c["not_json"] = "{not json"
    c["array_root"] = "[1, 2, 3]"
    c["empty"] = ""
    c["ws"] = "   "
    c["empty_obj"] = "{}"
    c["trailing_comma"] = doc(ev(0) + ",")
    c["single_quotes"] = "{'schema_version': 1}"
    c["leading_zero"] = doc(ev("01"))
    c["one_dot"] = doc(ev(0, start="1."))
    c["ctrl_char"] = doc(ev(0, name='"a\tb"'))
    c["bad_escape"] = doc(ev(0, name='"a\\xb"'))
    c["unterminated"] = doc(ev(0))[:-3]
    c["extra_data"] = doc(ev(0)) + " x"
    c["version_2"] = '{"schema_version": 2, "time_unit": "microseconds"}'
    c["version_str"] = '{"schema_version": "1", "time_unit": "microseconds"}'
    c["version_float"] = '{"schema_version": 1.0, "time_unit": "microseconds", "events": []}'
    c["version_true"] = '{"schema_version": true, "time_unit": "microseconds"}'
    c["version_missing"] = '{"time_unit": "microseconds"}'
    c["unit_seconds"] = '{"schema_version": 1, "time_unit": "seconds"}'
    c["unit_missing"] = '{"schema_version": 1}'
    c["keys_reordered"] = '{"events": [' + ev(0) + '], "time_unit": "microseconds", "schema_version": 1}'
    for k, v in enumerate(["null", "{}", '"x"', "5"]):
        c[f"events_type_{k}"] = "{" + HEAD + f', "events": {v}' + "}"
    c["events_dup_key"] = "{" + HEAD + ', "events": [' + ev(0) + '], "events": [' + ev(5) + ", " + ev(6, start=3) + "]}"
    c["events_dup_key_null"] = "{" + HEAD + ', "events": [' + ev(0) + '], "events": null}'
    c["no_events"] = "{" + HEAD + "}"
    c["event_not_obj"] = doc(ev(0) + ", 5, " + ev(1, start=9))
    c["first_error_wins"] = doc(", ".join([ev(0), ev(1, lane="bad"), ev("-3", start=5)]))
    c["syntax_after_schema"] = doc(ev(0, lane="bad")) + "}"
    c["version_before_events"] = '{"schema_version": 3, "time_unit": "microseconds", "events": [5]}'
    # -- duplicates / overlaps
    c["dup_ids"] = doc(", ".join([ev(0), ev(1, start=5), ev(0, start=9)]))
    c["dup_and_overlap"] = doc(", ".join([ev(0, dur=10), ev(1, start=5), ev(0, start=20)]))
    c["overlap"] = doc(", ".join([ev(0, dur=10), ev(1, start=5, dur=10)]))
    c["overlap_second_lane"] = doc(", ".join([ev(0, lane="cpu:1"), ev(1, lane="cpu:0", dur=10),
                                               ev(2, lane="cpu:0", start=5), ev(3, lane="cpu:1", start=0.5)]))
    c["overlap_two_lanes"] = doc(", ".join([ev(0, lane="cpu:1", dur=10), ev(1, lane="cpu:1", start=5),
                                             ev(2, lane="cpu:0", dur=10), ev(3, lane="cpu:0", start=5)]))
    c["zero_dur_no_overlap"] = doc(", ".join([ev(0, dur=0), ev(1, dur=1)]))
    c["unsorted_lane"] = doc(", ".join([ev(5, start=10), ev(3, start=0), ev(4, start=5)]))
    c["overlap_then_marker_err"] = doc(", ".join([ev(0, dur=10), ev(1, start=5)]), markers="5")
    # -- markers
    mk = lambda layer, ph, lane, s, e: f'{{"layer": {layer}, "phase": "{ph}", "cpu_lane": "{lane}", "start": {s}, "end": {e}}}'
    good = ", ".join([mk('"conv1"', "Forward", "cpu:0", 0, 5), mk('"conv2"', "Forward", "cpu:0", 4, 9),
                      mk('"*"', "Backward", "cpu:3", 0, 100), mk("7", "WeightUpdate", "cpu:0", 1.5, 2.5)])
    c["markers_ok"] = doc(ev(0, dur=10), markers=good)
    c["markers_not_list"] = doc(ev(0), markers=None) [:-1] + ', "layer_markers": {}}'
    c["marker_not_obj"] = doc(ev(0), markers="1")
    c["marker_phase_bad"] = doc(ev(0), markers=mk('"a"', "Sideways", "cpu:0", 0, 1))
    c["marker_gpu_lane"] = doc(ev(0), markers=mk('"a"', "Forward", "gpu:0:1", 0, 1))
    c["marker_start_end"] = doc(ev(0), markers=mk('"a"', "Forward", "cpu:0", 1, 1))
    c["marker_missing_layer"] = doc(ev(0), markers='{"phase": "Forward", "cpu_lane": "cpu:0", "start": 0, "end": 1}')
    c["marker_overlap"] = doc(ev(0, dur=10), markers=", ".join([mk('"c"', "Forward", "cpu:0", 0, 5),
                                                                 mk('"c"', "Forward", "cpu:0", 4, 9)]))
    c["marker_overlap_unsorted"] = doc(ev(0, dur=10), markers=", ".join([mk('"c"', "Forward", "cpu:0", 6, 9),
                                                                          mk('"d"', "Forward", "cpu:0", 0, 9),
                                                                          mk('"c"', "Forward", "cpu:0", 0, 7)]))
    c["marker_overlap_other_lane_ok"] = doc(ev(0, dur=10), markers=", ".join([mk('"c"', "Forward", "cpu:0", 0, 5),
                                                                               mk('"c"', "Forward", "cpu:1", 4, 9)]))
    # -- buckets / metadata
    gb = '"gradient_buckets": {"bucket_of_layer": {"l1": 0, "l2": 1}, "bucket_size_bytes": {"0": 100, "1": 5}}'
    c["buckets_ok"] = doc(ev(0), extra=gb)
    c["buckets_null"] = doc(ev(0), extra='"gradient_buckets": null')
    c["buckets_not_obj"] = doc(ev(0), extra='"gradient_buckets": 5')
    c["buckets_missing"] = doc(ev(0), extra='"gradient_buckets": {"bucket_of_layer": {}}')
    c["buckets_zero"] = doc(ev(0), extra='"gradient_buckets": {"bucket_of_layer": {}, "bucket_size_bytes": {"0": 0}}')
    c["buckets_unknown"] = doc(ev(0), extra='"gradient_buckets": {"bucket_of_layer": {"a": 3}, "bucket_size_bytes": {"0": 4}}')
    c["metadata_ok"] = doc(ev(0), extra='"metadata": {"a": 1, "b": "x", "c": [1, 2], "d": null}')
    c["metadata_bad"] = doc(ev(0), extra='"metadata": [1]')
    c["buckets_before_metadata"] = doc(ev(0), extra='"metadata": 5, "gradient_buckets": 5')
    c["marker_before_buckets"] = doc(ev(0), markers="1", extra='"gradient_buckets": 5')
    return c


def main():
    out = []
    for name, text in cases().items():
        rec = {"name": name, "text": text}
        try:
            d = parse_trace(text)
            rec["doc"] = document_to_object(d)
            rec["metadata"] = d.metadata
            rec["events_ns"] = [[e.id, e.start, e.duration] for e in d.events]
        except OverlapViolation as e:
            rec["error"] = e.name
            rec["message"] = e.message
            rec["ids"] = sorted([e.first_id, e.second_id])
        except KernsimError as e:
            rec["error"] = e.name
            rec["message"] = e.message
        except Exception as e:  # noqa: BLE001
            rec["error"] = f"<non-kernsim:{type(e).__name__}>"
        out.append(rec)
    with gzip.open(OUT, "wt") as f:
        json.dump(out, f)
    print(f"wrote {len(out)} cases to {OUT}")


if __name__ == "__main__":
    main()
