"""Merge one ncu capture's DRAM traffic into profiles/traffic.json:
    python tools/traffic_json.py profiles/traffic.json <model> <step> <rep.ncu-rep>"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import summary  # noqa: E402


def to_bytes(v: str) -> float:
    num, _, unit = v.partition(" ")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit.strip(), 1)
    return float(num.replace(",", "")) * scale


def main():
    out, model, step, rep = sys.argv[1:5]
    rows = summary(rep)
    if not rows:
        return
    d = rows[0]
    rd = to_bytes(d["dram__bytes_read.sum"])
    wr = to_bytes(d["dram__bytes_write.sum"])
    p = Path(out)
    data = json.loads(p.read_text()) if p.exists() else {}
    data.setdefault(model, {})[step] = {
        "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
        "duration": d.get("gpu__time_duration.sum"), "kernel": d.get("kernel"),
        "tensor_pipe_pct": d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "source": f"ncu --set full, {Path(rep).name}"}
    p.write_text(json.dumps(data, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
