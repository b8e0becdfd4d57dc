"""Summaries of ncu CSV exports: launch lists (per-kernel mean of each
metric) and raw pages (stall reasons, pipes, occupancy, dram bytes)."""
import collections
import csv
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    names = {}
    for r in rows[hi + 1:]:
        k = r[ki].split('(')[0][:48]
        names[r[ii]] = k
        agg[k][r[mi]] += float(r[vi].replace(',', ''))
    c = collections.Counter(names.values())
    tot = sum(d.get('gpu__time_duration.sum', 0) for d in agg.values())
    for k, d in sorted(agg.items(), key=lambda kv: -kv[1].get('gpu__time_duration.sum', 0)):
        t = d.get('gpu__time_duration.sum', 0)
        extra = " ".join(f"{m.split('__')[1][:16]}={v / c[k]:.4g}" for m, v in d.items() if 'time' not in m)
        print(f"{k:48s} n={c[k]:4d} total={t / 1e6:9.3f} ms ({t / tot:5.1%}) per={t / c[k] / 1e3:9.1f} us {extra}")


def raw(path):
    rows = list(csv.reader(open(path)))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    st = [(k, d[k]) for k in h if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')]
    st.sort(key=lambda kv: -float(kv[1].replace(',', '') or 0))
    print("stalls/issue:", ", ".join(f"{k[34:-23]}={float(x):.2f}" for k, x in st[:8]))
    # executed FP64 thread instructions (predicated-on lanes only), to set
    # against the algorithmic work model of bench.work_counts
    try:
        cyc = float(d['smsp__cycles_elapsed.avg'].replace(',', ''))
        fp = {op: float(d[f'smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed'].replace(',', '')) * cyc
              for op in ('dadd', 'dmul', 'dfma')}
        print("  fp64 thread instr: " + ", ".join(f"{k}={v:.4g}" for k, v in fp.items())
              + f", total={sum(fp.values()):.4g}")
    except (KeyError, ValueError):
        pass
    for key in ['gpu__time_duration.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
                'sm__warps_active.avg.per_cycle_active', 'launch__registers_per_thread', 'launch__grid_size',
                'launch__block_size', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
                'smsp__issue_active.avg.pct_of_peak_sustained_active', 'lts__t_sector_hit_rate.pct',
                'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__occupancy_limit_registers',
                'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'dram__throughput.avg.pct_of_peak_sustained_elapsed']:
        if key in d:
            print(f"  {key} = {d[key]} {units[h.index(key)]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        (launches if 'launch' in p else raw)(p)
