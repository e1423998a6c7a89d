"""ncu --set full capture -> the traffic record bench.py reads (profiles/rNN_traffic*.json).

    python scripts/ncu_to_traffic.py rep.ncu-rep "source command" out.json
Per kernel in the report: duration, DRAM bytes read/written, L2 hit rate, pipe utilisation, SM clock.
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {"time_ms": "gpu__time_duration.sum", "dram_bytes_read": "dram__bytes_read.sum",
           "dram_bytes_write": "dram__bytes_write.sum",
           "dram_pct_of_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "l2_hit_pct": "lts__t_sector_hit_rate.pct",
           "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm_clock_ghz": "gpc__cycles_elapsed.avg.per_second"}
SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "%": 1.0, "Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9}


def main(rep, source, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    kernels = {}
    for r in rows[2:]:
        rec = {}
        for k, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                rec[k] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
        kernels[r[hdr.index("Kernel Name")]] = rec
    json.dump({"source": source, "kernels": kernels}, open(out, "w"), indent=1)
    print(json.dumps(kernels, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
