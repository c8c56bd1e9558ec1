#!/usr/bin/env python3
"""Summarise an FI_TC_TRACE timeline (last launch in the file): per-CTA unit
spans (producer start -> MMA done -> epilogue ready -> epilogue done), the
kernel span, and when CTAs go idle."""
import statistics
import sys


def main(path):
    launches, cur = [], None
    for line in open(path):
        if line.startswith("launch"):
            cur = {"hdr": line.strip(), "rows": []}
            launches.append(cur)
        elif line.startswith("wait"):  # FI_TC_WAITPROF builds: cta full_wait mma_loop empty_wait prod_loop kb
            cur.setdefault("wait", []).append([int(x) for x in line.split()[1:]])
        elif cur is not None:
            vals = [int(x) for x in line.split()]
            cur["rows"].append(tuple(vals[:6]))
            if len(vals) >= 10 and vals[8]:  # tail fixup: published, peers staged, drained
                cur.setdefault("fix", []).append((vals[4], vals[8], vals[9], vals[5]))
                if len(vals) >= 11 and vals[10]:
                    cur.setdefault("drain", []).append((vals[10] - vals[4], vals[8] - vals[10]))
                if len(vals) >= 13 and vals[12] and vals[11]:
                    cur.setdefault("drain_clk", []).append(vals[12] - vals[11])
            # prologue stamps (slot 7 of units 0..2): entry, TMEM alloc done, prologue synced
            if len(vals) >= 14 and vals[13] and vals[1] == 0:
                cur.setdefault("entry", []).append((vals[13], vals[2]))
            if len(vals) >= 14 and vals[13] and vals[1] in (1, 2, 3, 4):
                cur.setdefault("pro%d" % vals[1], {})[vals[0]] = vals[13]
            if len(vals) >= 8 and vals[6] and vals[7] and vals[3] > vals[2]:
                cur.setdefault("mhz", []).append((vals[7] - vals[6]) / (vals[3] - vals[2]) * 1e3)
    last = launches[-1]
    rows = last["rows"]
    if last.get("mhz"):
        print(f"effective SM clock (clock64 / globaltimer over MMA spans): median "
              f"{statistics.median(last['mhz']):.0f} MHz, min {min(last['mhz']):.0f}, max {max(last['mhz']):.0f}")
    t0 = min(r[2] for r in rows if r[2])
    end = max(max(r[3], r[5]) for r in rows)
    print(last["hdr"], f"span {(end - t0) / 1e3:.1f} us, {len(set(r[0] for r in rows))} CTAs")
    if last.get("entry"):
        e0 = min(e for e, _ in last["entry"])
        lag = [(p - e) / 1e3 for e, p in last["entry"] if p]
        print(f"kernel entry: CTAs enter over {(max(e for e, _ in last['entry']) - e0) / 1e3:.2f} us; entry -> first "
              f"TMA load median {statistics.median(lag):.2f} us, max {max(lag):.2f}; first entry -> last stamp "
              f"{(end - e0) / 1e3:.1f} us")
        ent = {c: e for c, (e, _) in zip([r[0] for r in rows if r[1] == 0], last["entry"])}
        for key, what in (("pro1", "TMEM alloc done"), ("pro2", "prologue cluster sync done"),
                          ("pro3", "C stores complete"), ("pro4", "TMEM dealloc done (exit)")):
            d = [(t - ent[c]) / 1e3 for c, t in last.get(key, {}).items() if c in ent]
            if d:
                print(f"  entry -> {what}: median {statistics.median(d):.2f} us, max {max(d):.2f}")
    per_cta = {}
    for cta, unit, p0, m1, e2, e3 in rows:
        per_cta.setdefault(cta, []).append((unit, p0, m1, e2, e3))
    done = [max(u[4] for u in us) - t0 for us in per_cta.values()]
    print(f"CTA finish: min {min(done) / 1e3:.1f} us  median {statistics.median(done) / 1e3:.1f}  "
          f"max {max(done) / 1e3:.1f}")
    nunits = max(len(us) for us in per_cta.values())
    for i in range(nunits):
        mm = [(us[i][2] - us[i][1]) for us in per_cta.values() if len(us) > i and us[i][2] and us[i][1]]
        ep = [(us[i][4] - us[i][3]) for us in per_cta.values() if len(us) > i and us[i][4] and us[i][3]]
        st = [(us[i][1] - t0) for us in per_cta.values() if len(us) > i and us[i][1]]
        if mm:
            print(f"unit {i}: starts {min(st) / 1e3:6.1f}..{max(st) / 1e3:6.1f} us  producer->MMA done median "
                  f"{statistics.median(mm) / 1e3:6.2f} us  epilogue median {statistics.median(ep) / 1e3 if ep else 0:6.2f} us"
                  f" max {max(ep) / 1e3 if ep else 0:6.2f}  (n={len(mm)})")


    wt = last.get("wait")
    if wt:
        med = statistics.median
        per_kb = [(w[2] / w[5], w[1] / w[5], w[4] / w[3] * w[5] / w[5]) for w in wt if w[5]]
        print(f"wait profile (SM cycles, median over {len(wt)} CTAs): MMA loop {med([w[2] for w in wt if w[2]]):.0f}, "
              f"of which waiting on full barriers {med([w[1] for w in wt if w[2]]):.0f}; producer loop "
              f"{med([w[4] for w in wt if w[4]]):.0f}, waiting on empty barriers {med([w[3] for w in wt if w[4]]):.0f}; "
              f"K blocks {med([w[5] for w in wt if w[5]]):.0f}; MMA loop per K block "
              f"{med([x[0] for x in per_kb]):.0f}, full-wait per K block {med([x[1] for x in per_kb]):.0f}")
    fix = last.get("fix")
    if fix:
        pub = [(p - r) / 1e3 for r, p, _, _ in fix]
        stg = [(g - p) / 1e3 for _, p, g, _ in fix if g]
        fin = [(d - g) / 1e3 for _, _, g, d in fix if g and d]
        med = lambda x: statistics.median(x) if x else 0.0
        print(f"tail fixup (median / max us): acc ready->partial published {med(pub):.2f} / {max(pub):.2f}  "
              f"published->peers staged {med(stg):.2f} / {max(stg) if stg else 0:.2f}  "
              f"staged->stored {med(fin):.2f} / {max(fin) if fin else 0:.2f}  (n={len(fix)}, owners={len(stg)})")
        dc = last.get("drain_clk")
        if dc:
            print(f"  TMEM->SMEM drain in SM cycles (clock64): median {statistics.median(dc):.0f}, max {max(dc)}")
        dr = last.get("drain")
        if dr:
            print(f"  of which TMEM->SMEM drain {med([d[0] / 1e3 for d in dr]):.2f} us, "
                  f"bulk stores complete {med([d[1] / 1e3 for d in dr]):.2f} us (medians)")


if __name__ == "__main__":
    main(sys.argv[1])
