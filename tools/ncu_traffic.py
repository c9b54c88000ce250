"""Writes profiles/ncu_traffic.json from an ncu --set full report of the KSG kernel (development
tool): DRAM bytes per pair (dram__bytes_read + write), ALU-pipe warp-instructions per pair
(sm__inst_executed_pipe_alu % of peak x 2 per SM-cycle x SM cycles x 148), issue / ALU utilisation.
    python tools/ncu_traffic.py <report.ncu-rep> <pairs in the profiled launch> <source note>"""
import csv
import io
import json
import os
import subprocess
import sys

rep, pairs, note = sys.argv[1], int(sys.argv[2]), sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2]


def m(name):
    return float(v[h.index(name)].replace(",", ""))


def bytes_of(name):
    unit = rows[1][h.index(name)]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    return m(name) * scale


alu_pct = m("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active")
cycles = m("sm__cycles_elapsed.avg")
d = {"ksg_kernel": v[h.index("Kernel Name")][:80],
     "ksg_dram_bytes_per_pair": round((bytes_of("dram__bytes_read.sum") + bytes_of("dram__bytes_write.sum")) / pairs),
     "alu_warp_instr_per_pair": round(alu_pct / 100 * 2 * cycles * 148 / pairs),
     "alu_pipe_pct": round(alu_pct, 1),
     "issue_active_pct": round(m("smsp__issue_active.avg.pct_of_peak_sustained_active"), 1),
     "warp_instr_per_pair": round(m("smsp__inst_executed.sum") / pairs),
     "algorithmic_bytes_per_pair": 12000,
     "source": note}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
json.dump(d, open(path, "w"), indent=1)
print(d)
