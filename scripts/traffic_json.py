"""profiles/<round>/traffic.json from the `ncu --set full` raw pages that
scripts/gpu_evidence.sh captures: DRAM bytes and duration per launch of each
profiled kernel, keyed "<kernel> | <workload>" as bench.committed_traffic
looks them up."""
import csv
import json
import sys

CAPTURES = [  # (raw csv, kernel, workload, details csv named in "source")
    ("mgs", "k_mgs_flow", "F(1024,1024,32) complex qd 1024x1024"),
    ("tree", "k_mono_tree_tma", "F(1024,1024,32) complex qd 1024x1024"),
    ("seg", "k_segments", "F(1024,1024,32) complex qd 1024x1024"),
    ("bsub", "k_backsub_look", "F(1024,1024,32) complex qd 1024x1024"),
    ("tail", "k_mgs_tail", "F(1024,1024,32) complex qd 1024x1024"),
    ("pipe", "k_mgs_pipe", "F(1024,1024,32) complex dd 1024x1024"),
    ("piped", "k_mgs_pipe", "F(1024,1024,32) complex d 1024x1024"),
    ("rows", "k_eval_rows", "F(1024,1024,32) complex d 1024x1024"),
    ("solve", "k_solve_batch", "C5 296 slots F(256,256,32) complex dd"),
]


def main(src, dst, tag):
    out = {}
    for name, kernel, workload in CAPTURES:
        try:
            rows = list(csv.reader(open(f"{src}/{name}_raw.csv")))
        except OSError:
            continue
        h, units, v = rows[0], rows[1], rows[2]
        d = dict(zip(h, v))
        u = dict(zip(h, units))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale[u["dram__bytes_read.sum"]]
        wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale[u["dram__bytes_write.sum"]]
        out[f"{kernel} | {workload}"] = {
            "dram_read_bytes": rd, "dram_write_bytes": wr,
            "duration": f"{d['gpu__time_duration.sum']} {u['gpu__time_duration.sum']}",
            "source": f"ncu --set full, profiles/{tag}/final/raw/{name}_raw.csv"}
    json.dump(out, open(dst, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
