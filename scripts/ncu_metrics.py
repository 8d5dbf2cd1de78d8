"""Print the key metrics of every kernel in an ncu report (ncu -i ... --page raw --csv)."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "smsp__inst_executed.sum", "launch__grid_size",
        "launch__registers_per_thread", "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def main(path, extra=()):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print("----", d.get("Kernel Name", "")[:60], "grid", d.get("Grid Size"), "block", d.get("Block Size"))
        for w in list(WANT) + list(extra):
            for h, u in zip(hdr, units):
                if h == w:
                    print(f"  {w} = {d[h]} {u}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
