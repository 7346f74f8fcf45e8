"""Summarise an ncu report: key raw metrics + top source lines by stall samples."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed"]
for i, name in enumerate(h):
    if name in want:
        print(f"{name:80s} {v[i]} {rows[1][i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f, res = None, []
for r in csv.reader(src.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 5 and r[0] not in ("", "Line No", "Function Name") and r[2] == "-":
        try:
            res.append((float(r[4]), f, r[0], r[1][:96]))
        except ValueError:
            pass
tot = sum(x[0] for x in res)
print("stall samples", tot)
for x in sorted(res, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print("%6.0f %5.1f%% %s:%s %s" % (x[0], 100 * x[0] / tot, x[1], x[2], x[3]))
