"""Summarise an event trace of the W = 32 tensor-core kernel (development aid).

    scripts/build_variant.sh trace -DMWB_TCH_TRACE
    MWB_TCH_TRACE_FILE=gpurun_out/tch_trace.txt MWB_LIB=$PWD/exp/libmwb_trace.so python scripts/tc_step_timing.py
    python scripts/tch_trace_report.py gpurun_out/tch_trace.txt

Events (CTA 0, clock64): 1 issuer saw step t's operands, 2 issuer got TMEM
back for item n, 3 / 4 a builder group started / published step t, 5..8 the
epilogue's accumulator wait, TMEM drain, partials barrier and outputs, 9 the
operand producer issued step t's A copy.  Tracing slows the traced CTA; read
the ratios, not the absolute cycles.
"""
import collections
import statistics
import sys


def main(path: str) -> None:
    ev = sorted(tuple(map(int, line.split())) for line in open(path))
    t0 = ev[0][0]
    ofull, acc_empty, a_issue, bstart, barr = {}, {}, {}, {}, {}
    epi = collections.defaultdict(dict)
    for tm, code, arg in ev:
        if code == 1:
            ofull[arg] = tm
        elif code == 2:
            acc_empty[arg] = tm
        elif code == 9:
            a_issue[arg] = tm
        elif code == 3:
            bstart[arg & 0xFFFFF] = tm
        elif code == 4:
            barr[arg & 0xFFFFF] = tm
        elif code in (5, 6, 7, 8):
            epi[arg & 0xFFFFF][(code, arg >> 20)] = tm
    steps = sorted(ofull)
    gaps = [ofull[steps[k + 1]] - ofull[steps[k]] for k in range(len(steps) - 1)]
    print(f"items {len(acc_empty)}  steps {len(steps)}  median step gap {statistics.median(gaps):.0f} clk")
    big = [g for g in gaps if g > 3 * statistics.median(gaps)]
    print(f"item-boundary gaps: {len(big)}, median {statistics.median(big) if big else 0:.0f} clk")
    for it in sorted(epi)[2:5]:
        e = epi[it]
        g0 = {code: tm - t0 for (code, grp), tm in e.items() if grp == 0}
        print(f"item {it}: acc_full {g0.get(5)}  drained +{g0.get(6, 0) - g0.get(5, 0)}  "
              f"partials +{g0.get(7, 0) - g0.get(6, 0)}  outputs +{g0.get(8, 0) - g0.get(7, 0)}")
    lat = [barr[t] - bstart[t] for t in barr if t in bstart]
    print(f"builder step latency: median {statistics.median(lat):.0f} clk")


if __name__ == "__main__":
    main(sys.argv[1])
