"""Write profiles/traffic.json from `ncu --set full` reports of the product
kernel (dev tool): dram__bytes_read.sum + dram__bytes_write.sum per launch,
keyed by workload and stamped with build.source_hash() so bench.py only
reports traffic captured from the kernel source it runs.

    python scripts/ncu_traffic.py config3=gpurun_out/r02_c3.ncu-rep config4=...
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2011_11880_b200.build import source_hash  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out_path = ROOT / "profiles" / "traffic.json"
data = json.loads(out_path.read_text()) if out_path.exists() else {}
data["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the product kernel "
                "k_eval_staged, from `ncu --set full -k regex:k_eval_staged` of scripts/kbench.py; "
                "source_hash identifies the kernel source (paper_2011_11880_b200/build.py)")
for arg in sys.argv[1:]:
    wl, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = lambda k: float(vals[hdr.index(k)]) * UNIT.get(units[hdr.index(k)], 1)
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    data[wl] = {"kernel": vals[hdr.index("Kernel Name")][:120], "bytes": int(rd + wr),
                "read": int(rd), "write": int(wr),
                "duration_us": get("gpu__time_duration.sum") / (1e3 if units[hdr.index(
                    "gpu__time_duration.sum")] == "nsecond" else 1),
                "report": Path(rep).name, "source_hash": source_hash()}
out_path.write_text(json.dumps(data, indent=1) + "\n")
print(json.dumps(data, indent=1))
