"""Key metrics + stall breakdown of one kernel from an ncu report (read here,
no GPU needed):

    python tools/ncu_summary.py gpurun_out/r01_decode.ncu-rep "<ncu command line>" > profiles/r01_ncu_decode_kernel.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "sm__icc_request_hit_rate.pct",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size", "launch__cluster_dim_x",
    "launch__shared_mem_per_block_dynamic",
    # tcgen05: tensor-memory / tensor-core shared-memory traffic and pipes
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
    "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def main(rep, cmd):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(head)}
    print(cmd)
    print("kernel:", vals[col["Kernel Name"]] if "Kernel Name" in col else "?")
    for k in KEYS:
        if k in col:
            print(f"{k:<70} {vals[col[k]]:>22} {units[col[k]]}")
    stalls = {h[len(STALL):]: float(vals[i].replace(",", "") or 0) for h, i in col.items()
              if h.startswith(STALL) and not h.endswith("_not_issued")}
    tot = sum(stalls.values())
    if tot > 0:
        print("stall reasons (share of PC samples):")
        for r, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:9]:
            print(f"  {r:<22} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
