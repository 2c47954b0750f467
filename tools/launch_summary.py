"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import io
import sys

txt = open(sys.argv[1]).read()
lines = [l for l in txt.splitlines() if l.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = {}, {}
for r in rows[1:]:
    name = r[ki]
    name = name if len(name) < 90 else name[:90] + "..."
    v = float(r[vi].replace(",", ""))
    if r[ui] == "msecond":
        v *= 1e6
    elif r[ui] == "usecond":
        v *= 1e3
    tot[name] = tot.get(name, 0.0) + v
    cnt[name] = cnt.get(name, 0) + 1
all_ns = sum(tot.values())
print(f"{'total us':>10} {'launches':>8} {'avg us':>9} {'share':>6}  kernel")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v / 1e3:10.1f} {cnt[k]:8d} {v / 1e3 / cnt[k]:9.2f} {100 * v / all_ns:5.1f}%  {k}")

# per-kernel launch-duration histogram (full-class launches vs the streamed host apply's per-stage launches)
durs = {}
for r in rows[1:]:
    name = r[ki] if len(r[ki]) < 90 else r[ki][:90] + "..."
    v = float(r[vi].replace(",", ""))
    v = v * 1e6 if r[ui] == "msecond" else (v * 1e3 if r[ui] == "usecond" else v)
    durs.setdefault(name, []).append(v / 1e3)
for k, ds in sorted(durs.items(), key=lambda kv: -sum(kv[1])):
    ds = sorted(ds)
    big = [d for d in ds if d >= 0.5 * ds[-1]]
    print(f"{k[:60]}: {len(big)} launches >= half the longest, median {big[len(big) // 2]:.1f} us; "
          f"{len(ds) - len(big)} shorter (median {ds[(len(ds) - len(big)) // 2]:.1f} us)" if len(ds) > len(big)
          else f"{k[:60]}: {len(ds)} launches, median {ds[len(ds) // 2]:.1f} us")
