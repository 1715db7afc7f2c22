"""Summarise the per-tile prefill timeline (tools/pf_trace.sh, a -DKB_PF_TRACE
build): median cycles of each hop between a softmax warpgroup publishing P
and its next S, over the steady-state tiles of one CTA.

    python tools/pf_trace_report.py gpurun_out/pft.log
"""
import statistics as st
import sys

rows = [list(map(int, l.split()[1:])) for l in open(sys.argv[1]) if l.startswith("pft")]
rows = rows[-256:]  # the last launch
d = {(r[0], r[1]): r[2:] for r in rows}
J = max(j for j, _ in d)


def med(f):
    return st.median(f(j, t) for j in range(20, J - 20) for t in (0, 1))


out = {
    "softmax S -> p_lo": med(lambda j, t: d[(j, t)][1] - d[(j, t)][0]),
    "softmax p_lo -> p_hi": med(lambda j, t: d[(j, t)][2] - d[(j, t)][1]),
    "p_lo published -> MMA sees it": med(lambda j, t: d[(j, t)][3] - d[(j, t)][1]),
    "PV_lo issue (blocking)": med(lambda j, t: d[(j, t)][4] - d[(j, t)][3]),
    "p_hi published -> MMA sees it": med(lambda j, t: d[(j, t)][5] - d[(j, t)][2]),
    "PV_hi issue (blocking)": med(lambda j, t: d[(j, t)][6] - d[(j, t)][5]),
    "PV_hi issued -> QK(j+1) issued": med(lambda j, t: d[(j + 1, t)][7] - d[(j, t)][6]),
    "QK(j+1) issued -> S(j+1) seen": med(lambda j, t: d[(j + 1, t)][0] - d[(j + 1, t)][7]),
    "p_hi -> S(j+1) (softmax idle)": med(lambda j, t: d[(j + 1, t)][0] - d[(j, t)][2]),
    "period per tile": med(lambda j, t: d[(j + 1, t)][0] - d[(j, t)][0]),
}
for k, v in out.items():
    print(f"{k:34s} {v:8.0f} cycles")
