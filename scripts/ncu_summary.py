"""Condense an `ncu --set full` report (raw page CSV) into the metrics the roofline uses."""
import csv, json, subprocess, sys

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1e-9),
    "tensor_pipe_active_pct": ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
    "tensor_mem_active_pct": ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_read_bytes": ("lts__t_sectors_op_read.sum", 32),
    "l2_write_bytes": ("lts__t_sectors_op_write.sum", 32),
    "l2_bytes": ("lts__t_bytes.sum", 1),
    "smem_pipe_pct": ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_elapsed", 1),
    "l1tex_throughput_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
}
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "msecond": 1e6, "usecond": 1e3, "nsecond": 1,
        "ms": 1e6, "us": 1e3, "ns": 1, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def main(rep, out_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, (m, scale) in KEYS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", "")) * UNIT.get(units[i], 1) * scale
                except ValueError:
                    v = r[i]
                d[k] = round(v, 4) if isinstance(v, float) else v
        res.append(d)
    for d in res:
        print(json.dumps(d))
    if out_json:
        json.dump(res, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
