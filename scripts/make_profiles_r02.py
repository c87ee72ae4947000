"""Summarises round-2 ncu captures (gpurun_out/prof02b_<scene>.ncu-rep) into
profiles/: a metrics summary per scene, the per-source-line profile, and the
per-launch DRAM traffic / instruction counts bench.py reads
(profiles/k1_traffic.json, profiles/k1_instructions.json).  Dev aid.
usage: python scripts/make_profiles_r02.py scene:rays [scene:rays ...]"""
import csv, io, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def num(v):
    return float(str(v).replace(",", ""))


traffic_path = os.path.join(P, "k1_traffic.json")
inst_path = os.path.join(P, "k1_instructions.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
inst = json.load(open(inst_path)) if os.path.exists(inst_path) else {}
for arg in sys.argv[1:]:
    scene, rays = arg.split(":")
    rays = float(rays)
    rep = os.path.join(ROOT, "gpurun_out", f"prof02b_{scene}.ncu-rep")
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                          capture_output=True, text=True).stdout
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines.py"), rep,
                            str(rays), "40"], capture_output=True, text=True).stdout
    v, u = raw(rep)
    dr = num(v["dram__bytes_read.sum"]) * (1e6 if u["dram__bytes_read.sum"] == "Mbyte" else
                                            1e9 if u["dram__bytes_read.sum"] == "Gbyte" else
                                            1e3 if u["dram__bytes_read.sum"] == "Kbyte" else 1)
    dw = num(v["dram__bytes_write.sum"]) * (1e6 if u["dram__bytes_write.sum"] == "Mbyte" else
                                             1e9 if u["dram__bytes_write.sum"] == "Gbyte" else
                                             1e3 if u["dram__bytes_write.sum"] == "Kbyte" else 1)
    wi = num(v["smsp__inst_executed.sum"])
    # thread instructions: the source page's per-line sum (ncu_lines.py, first line)
    ti = float(lines.split("thread instr per unit ")[1].split(";")[0]) * rays
    with open(os.path.join(P, f"r02_k1_{scene}_ncu_summary.txt"), "w") as f:
        f.write(f"# ncu --set full, one K1 launch of `scripts/run_scene.py {scene}` ({rays:.3g} rays)\n")
        f.write(summ)
        f.write(f"dram bytes per launch {dr + dw:.4g} (read {dr:.4g}, write {dw:.4g})\n")
        f.write(f"warp instructions per ray {wi / rays:.2f}, thread instructions per ray {ti / rays:.1f}\n")
        f.write("\n# per CUDA source line (scripts/ncu_lines.py)\n" + lines)
    traffic[scene] = {"dram_bytes_per_launch": dr + dw, "rays_per_launch": rays,
                      "source": f"profiles/r02_k1_{scene}_ncu_summary.txt"}
    inst[scene] = {"warp_inst_per_ray": wi / rays, "thread_inst_per_ray": ti / rays,
                   "source": f"profiles/r02_k1_{scene}_ncu_summary.txt"}
    print(scene, f"dram {dr + dw:.4g} B, {wi / rays:.2f} warp-inst/ray")
json.dump(traffic, open(traffic_path, "w"), indent=1)
json.dump(inst, open(inst_path, "w"), indent=1)
