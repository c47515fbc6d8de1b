"""Print the last step's kernels from an ncu --metrics gpu__time_duration.sum
CSV launch list: python scripts/launch_table.py FILE [steps_in_file]."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
k, mv, g = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
items = [(r[k][:80], float(r[mv].replace(",", "")) / 1000, r[g]) for r in rows[start + 1:]
         if r[h.index("Metric Name")] == "gpu__time_duration.sum"]
# the step is the tail 1/steps of the launches that repeat
n = len(items) // steps
last = items[-n:]
for name, us, grid in last:
    print(f"{us:8.1f}  {name}  {grid}")
print(f"total {sum(x[1] for x in last):.1f} us, {len(last)} kernels")
