#!/usr/bin/env python3
"""supercell S x tile drift halo h x sort interval K sweep
with a per-stage breakdown in the shape of the paper's Tables 5/6
(supercell sizes chosen so the supercell's grid data fit
on-chip; time per stage).  The GPU analogue of the paper's cache model is the
shared-memory footprint of one CTA's E/B and J tiles, (S + 2h + 2)^3 x 6 fp64
plus (S + 2h + 3)^3 x 9 u32 (padded), which also sets the CTAs per SM.

One process per workload; particles are generated once and every
configuration runs in a fresh context (5 warm-up steps, then `steps` timed
with CUDA events on the library stream, plus a profiled pass of the same
steps for the stage split).  Prints a markdown table; run under gpurun:
    python tools/sweep.py C3 40 > profiles/r02/sweep_S_h_K_C3.md
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1608_01009_b200 as pkg  # noqa: E402
from synth import gen_particles, get_config  # noqa: E402


def tile_smem_kb(S, h):
    """Shared bytes of one CTA's tiles (push_tile.cu TileGeom, S >= 4 pitches)."""
    te, tj = S + 2 * h + 2, S + 2 * h + 3
    def up(v, m, r):
        return v + ((r - v % m) % m + m) % m
    epx = up(te, 8, 4) if S >= 4 else te
    jpx = up(tj, 8, 4) if S >= 4 else tj
    jpy = up(jpx * tj, 32, 16) if S >= 4 else jpx * tj
    return (6 * epx * te * te * 8 + 9 * jpy * tj * 4) / 1024


def run(wl, parts, steps):
    n = sum(p.shape[1] for p, _ in parts)
    out = {}
    for flags in (0, pkg.FLAG_PROFILE):
        sim = pkg.simulation_from_workload(wl, capacity_factor=1.0, flags=flags)
        for s, (P, ids) in enumerate(parts):
            sim.set_particles(s, P, ids)
        sim.step(5)
        if flags:
            sim.stage_times()
            sim.step(steps)
            st = sim.stage_times()
            out["stage"] = {k: st[k] / steps for k in ("sort", "particle", "field")}
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(sim.stream)
            sim.step(steps)
            e1.record(sim.stream)
            torch.cuda.synchronize()
            out["gups"] = n * steps / (e0.elapsed_time(e1) * 1e-3) / 1e9
        sim.close()
        del sim
        torch.cuda.empty_cache()
    return out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    base = get_config(name)
    parts = gen_particles(base)
    print(f"# {name}: supercell S x halo h x sort interval K ({steps} timed steps after 5 warm-up)\n")
    print("| S | h | tile KB/CTA | K | G upd/s | ns/particle/step | particle ms/step | sort ms/step | field ms/step |")
    print("|---|---|---|---|---|---|---|---|---|")
    best = None
    for S in (4, 2):
        for h in (1, 2):
            for K in (5, 10, 20, 40):
                wl = base.with_(supercell=S, halo=h, sort_every=K)
                r = run(wl, parts, steps)
                st = r["stage"]
                print(f"| {S} | {h} | {tile_smem_kb(S, h):.0f} | {K} | {r['gups']:.2f} | {1.0 / r['gups']:.4f} | "
                      f"{st['particle']:.4f} | {st['sort']:.4f} | {st['field']:.4f} |", flush=True)
                if best is None or r["gups"] > best[0]:
                    best = (r["gups"], S, h, K)
    print(f"\nbest: S = {best[1]}, h = {best[2]}, K = {best[3]}: {best[0]:.2f} G upd/s")


if __name__ == "__main__":
    main()
