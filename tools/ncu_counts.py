#!/usr/bin/env python3
"""Fold one ncu --csv metric capture of the fused particle kernel into
profiles/ncu_particle_traffic.json (the `traffic` and counted-fp64 fields of
bench.py's roofline):

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,\
smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,\
smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,\
smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,\
l1tex__data_pipe_lsu_wavefronts.sum \
        --clock-control none -k regex:k_push_tile -s 3 -c 1 --csv \
        python tools/run_steps.py C3 6 > gpurun_out/ncu_counts_C3.csv
    python tools/ncu_counts.py C3 gpurun_out/ncu_counts_C3.csv COMMIT

fp64 flop of the launch = 2 DFMA + DADD + DMUL thread instructions; per
update = that / the particles of the launch (the workload's particle count:
one launch pushes every species at N = 1)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def read_metrics(path):
    rows = list(csv.reader(open(path)))
    hdr, out, kernel = None, {}, None
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            kernel = d["Kernel Name"]
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            out[d["Metric Name"]] = v * scale
    return kernel, out


def main():
    wl_name, path, commit = sys.argv[1], sys.argv[2], sys.argv[3]
    from synth import get_config
    wl = get_config(wl_name)
    kernel, m = read_metrics(path)
    n = wl.n_particles
    occ_cells = wl.nx * wl.ny * ((wl.plasma_z[1] - wl.plasma_z[0]) if wl.plasma_z else wl.nz)
    flop = (2 * m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
            + m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
            + m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"])
    p = os.path.join(ROOT, "profiles", "ncu_particle_traffic.json")
    data = json.load(open(p)) if os.path.exists(p) else {}
    data["_source"] = ("ncu --metrics (dram__bytes_read/write.sum, smsp__sass_thread_inst_executed_op_"
                       "d{fma,add,mul}_pred_on.sum) of one fused particle-kernel launch (step 3 after the "
                       "initial sort), --clock-control none; tools/ncu_counts.py")
    data[wl_name] = {
        "kernel": kernel.split("(")[0] if kernel else None,
        "commit": commit,
        "capture": os.path.basename(path),
        "bytes_per_launch": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
        "dram_read_bytes": m["dram__bytes_read.sum"],
        "dram_write_bytes": m["dram__bytes_write.sum"],
        "alg_bytes_per_launch": 96.0 * n + 72.0 * occ_cells,
        "fp64_flop_per_launch": flop,
        "fp64_flop_per_update": flop / n,
    }
    if "l1tex__data_pipe_lsu_wavefronts.sum" in m:
        # the L1/shared-memory data pipe: one 128-byte wavefront per SM clock
        data[wl_name]["lsu_wavefronts_per_launch"] = m["l1tex__data_pipe_lsu_wavefronts.sum"]
    json.dump(data, open(p, "w"), indent=1)
    print(json.dumps(data[wl_name], indent=1))


if __name__ == "__main__":
    main()
