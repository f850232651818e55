"""Extract the per-launch DRAM traffic of r2_allreduce_kernel from an
`ncu --set full` capture into the JSON file bench.py reads for
roofline.traffic (one capture per round: profiles/rNN_ncu_traffic.json).

    python tools/ncu_traffic.py gpurun_out/ev1/sim8_full.ncu-rep profiles/r02_ncu_traffic.json "<how it was captured>"
"""
import csv
import io
import json
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "": 1, "register/thread": 1}


def main(rep, out, how):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]

    def val(row, name):
        i = head.index(name)
        return float(row[i].replace(",", "")) * UNITS[units[i]]

    for row in rows[2:]:
        name = row[head.index("Kernel Name")]
        if "r2_allreduce_kernel" not in name and "r2_ring_kernel" not in name:
            continue
        rd, wr = val(row, "dram__bytes_read.sum"), val(row, "dram__bytes_write.sum")
        d = {"workload": "8 simulated ranks x 256 MiB bf16, K=8, W=2, 512 KiB chunks (bench.py N=1 default)",
             "kernel": name.split("(")[0].split("::")[-1],
             "dram_bytes_read_per_launch": int(rd), "dram_bytes_write_per_launch": int(wr),
             "dram_bytes_per_launch": int(rd + wr),
             "ncu_duration_ms": val(row, "gpu__time_duration.sum"),
             "grid": int(val(row, "launch__grid_size")),
             "registers_per_thread": int(val(row, "launch__registers_per_thread")),
             "source": how}
        with open(out, "w") as f:
            json.dump(d, f, indent=2)
            f.write("\n")
        print(json.dumps(d))
        return
    raise SystemExit("no r2_allreduce_kernel launch in " + rep)


if __name__ == "__main__":
    main(*sys.argv[1:4])
