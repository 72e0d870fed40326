"""Write a profiles/ summary of one ncu --set full report: the command, the kernel,
DRAM bytes per launch, then tools/ncu_summary.py's key metrics and stall breakdown.
usage: python tools/profile_txt.py rep.ncu-rep "<ncu args>" "<profiled command>" ["<what one launch is>"]
  > profiles/…"""
import csv
import io
import subprocess
import sys

rep, ncu_args, cmd = sys.argv[1:4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
names, units, vals = rows[0], rows[1], rows[2]
col = {n: i for i, n in enumerate(names)}


def val(n):
    v = vals[col[n]].replace(",", "")
    u = units[col[n]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return float(v) * scale, u


rd, _ = val("dram__bytes_read.sum")
wr, _ = val("dram__bytes_write.sum")
print(f"# ncu {ncu_args}")
print(f"#   {cmd}")
print("# one launch = " + (sys.argv[4] if len(sys.argv) > 4 else
                           "one 1352x1014 view of the C3 scene (300k Gaussians)"))
print(f"kernel: {vals[col['Kernel Name']][:90]}")
print(f"dram_bytes_per_launch: {int(rd + wr)}  (read {rd / 1e6:.3f} MB, write {wr / 1e6:.3f} MB)")
sys.stdout.flush()
subprocess.run([sys.executable, "tools/ncu_summary.py", rep])
