"""Instruction and stall shares of k_trace_query by code region (psg_query.cu
line ranges) from an ncu report: python tools/regions.py REP [events]."""
import csv
import subprocess
import sys

rep = sys.argv[1]
events = float(sys.argv[2]) if len(sys.argv) > 2 else 4.9982e9
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:k_trace_query",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname, hdr, res = None, None, []
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
    elif len(r) > 3 and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr):
        try:
            res.append((fname, int(r[0]), int(r[hdr.index("Instructions Executed")]),
                        int(r[hdr.index("Warp Stall Sampling (All Samples)")])))
        except ValueError:
            pass
ti = sum(x[2] for x in res) or 1
ts = sum(x[3] for x in res) or 1
src = open("paper_2605_03561_b200/csrc/psg_query.cu").read().splitlines()


def find(s, start=0):
    for i in range(start, len(src)):
        if s in src[i]:
            return i + 1
    raise KeyError(s)


marks = [("run_events (general path)", find("__device__ __forceinline__ void run_events")),
         ("run_events_il (general path)", find("__device__ __forceinline__ void run_events_il")),
         ("run_block", find("__device__ __forceinline__ void run_block")),
         ("helpers", find("__device__ __forceinline__ u64 cell64")),
         ("run_fast", find("__device__ __forceinline__ void run_fast(")),
         ("run_fast_il", find("__device__ __forceinline__ void run_fast_il")),
         ("flush_fast", find("__device__ __forceinline__ void flush_fast")),
         ("prologue", find("k_trace_query(query_params p) {")),
         ("chunk head", find("for (uint32_t c = c_lo;; ++c) {")),
         ("step: loads + window class", find("while (pos < E1) {")),
         ("step: fast-path setup", find("if (CUBE && kept && all && !cwide")),
         ("step: general setup", find("if (!done) {")),
         ("chunk flush (other)", find("// ---- phase 2")),
         ("epilogue", find("if (!active) return;", find("// ---- phase 2"))),
         ("end", len(src) + 1)]
print(f"total {ti} warp inst = {ti / events * 256:.0f} per 256-event step; stall samples {ts}")
for (name, a), (_, b) in zip(marks, marks[1:]):
    i = sum(x[2] for x in res if x[0] == "psg_query.cu" and a <= x[1] < b)
    s = sum(x[3] for x in res if x[0] == "psg_query.cu" and a <= x[1] < b)
    print(f"{name:30s} inst {100 * i / ti:5.1f}% ({i / events * 256:6.1f}/step)  stall {100 * s / ts:5.1f}%")
oth = {}
for x in res:
    if x[0] != "psg_query.cu":
        oth[x[0]] = oth.get(x[0], (0, 0))
        oth[x[0]] = (oth[x[0]][0] + x[2], oth[x[0]][1] + x[3])
for f, (i, s) in sorted(oth.items(), key=lambda kv: -kv[1][0]):
    print(f"{f:30s} inst {100 * i / ti:5.1f}% ({i / events * 256:6.1f}/step)  stall {100 * s / ts:5.1f}%")
