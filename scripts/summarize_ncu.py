"""Summaries of ncu outputs for profiles/: launch-list shares and --set full metrics."""
import collections, csv, json, re, subprocess, sys


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        v = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)  # -> us
        name = re.sub(r"\(.*", "", d["Kernel Name"])
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    return [{"kernel": k, "total_us": round(tot[k], 1), "share": round(tot[k] / T, 4), "launches": cnt[k],
             "avg_us": round(tot[k] / cnt[k], 2)} for k in sorted(tot, key=lambda k: -tot[k])]


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]
    res = []
    for r in rows[2:]:
        d = {w: r[hdr.index(w)] for w in want if w in hdr}
        st = [(hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i])) for i in range(len(hdr))
              if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled") and not hdr[i].endswith("not_issued")
              and r[i] not in ("", "n/a")]
        st.sort(key=lambda s: -s[1])
        d["top_stalls"] = st[:5]
        res.append(d)
    return res


if __name__ == "__main__":
    kind, path, out = sys.argv[1], sys.argv[2], sys.argv[3]
    data = launch_shares(path) if kind == "launches" else full_metrics(path)
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(data[:6], indent=1)[:3000])
