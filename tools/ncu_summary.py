"""Summarise ncu outputs into profiles/ (tracked).

  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.txt
  python tools/ncu_summary.py full gpurun_out/search_full.ncu-rep profiles/search_ncu.json \
        --config-key KEY --alg-bytes B --label r01

`launches`: per-kernel totals of gpu__time_duration.sum (cold-cache,
serialised: compare shares, not absolutes).
`full`: the key metrics of one `ncu --set full` capture (DRAM bytes per launch,
duration, L2 hit rate, occupancy, registers, smem) as JSON; bench.py reads
dram_bytes_per_launch from it as roofline.traffic when config_key matches.
"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
        "s": 1e3, "second": 1e3}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    agg, tot = {}, 0.0
    for r in rows[i + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ms = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1e-6)
        name = d["Kernel Name"].split("(")[0]
        a = agg.setdefault(name, [0.0, 0])
        a[0] += ms
        a[1] += 1
        tot += ms
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (source {src})",
             "# total_ms  launches  mean_ms  share  kernel"]
    for k, (ms, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        lines.append(f"{ms:12.3f} {c:5d} {ms / c:10.3f} {100 * ms / tot:6.2f}%  {k}")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, dst, key, alg, label, command=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    res = []
    for row in r[2:]:
        d = dict(zip(h, row))
        unit = dict(zip(h, u))

        def val(k, conv=None):
            v = float(d[k].replace(",", ""))
            if conv == "bytes":
                v *= BYTES.get(unit[k].split("/")[0], 1)
            if conv == "ms":
                v *= UNIT.get(unit[k], 1e-6)
            return v

        rd = val("dram__bytes_read.sum", "bytes")
        wr = val("dram__bytes_write.sum", "bytes")
        ms = val("gpu__time_duration.sum", "ms")
        res.append({
            "kernel": d["Kernel Name"].split("(")[0],
            "duration_ms": ms,
            "dram_read_bytes": rd, "dram_write_bytes": wr,
            "dram_bytes_per_launch": rd + wr,
            "dram_GBps": (rd + wr) / (ms * 1e-3) / 1e9,
            "l2_hit_rate_pct": val("lts__t_sector_hit_rate.pct"),
            "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers_per_thread": val("launch__registers_per_thread"),
            "smem_per_block_bytes": val("launch__shared_mem_per_block", "bytes"),
            "grid": val("launch__grid_size"), "block": val("launch__block_size"),
            "sm_throughput_pct": val("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        })
        if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active" in d:
            res[-1]["tensor_pipe_active_pct"] = val(
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
    top = res[0]
    top.update({"config_key": key, "label": label, "source": rep,
                "algorithmic_bytes_per_launch": alg,
                "command": command or ("ncu --set full --clock-control none --import-source on "
                                       "-k regex:search_kernel -s 3 -c 1 python bench.py "
                                       "--steps 1 --warmup 3 --no-cpu")})
    json.dump(top, open(dst, "w"), indent=1)
    print(json.dumps(top, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        a = sys.argv[4:]
        kw = dict(zip(a[0::2], a[1::2]))
        full(sys.argv[2], sys.argv[3], kw.get("--config-key", ""),
             float(kw.get("--alg-bytes", "0")), kw.get("--label", ""), kw.get("--command"))
