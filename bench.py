"""Benchmark of the hot path (Algorithm 1 lines 3-7 for every level).

Headline workload: BASELINE.json configs[4] = config 5, the largest config (3D 256³, ε = 1/32,
contrast 1e3, L = 4, η = 2, 17³ = 4913 macropoints, 2 continua, 8 cell problems per macropoint) and
the north star's scaling config.  BASELINE.json's metric names no config, so the largest one is
the headline; `--config 2..4` runs the others (their per-level numbers are also printed beside the
headline under "other_configs").

One "step" = mch_solve_level(1..L) + mch_effective_coeffs on the device-resident medium: every
macropoint of every level, all N(1+d) cell problems, the Eq. (7) reductions.
value = cell-problem solves / s of the whole job (all ranks).  `e2e` repeats the step through the
C ABI with HOST buffers on an already planned context: mch_set_medium from pinned host κ/ψ (H2D
inside the timed region), the levels, mch_effective_coeffs into a pinned host buffer (D2H).

  python bench.py [--gpus N --steps K --warmup W --config C --impl {mch,reference}]

With --gpus N > 1 outside torchrun the script re-launches itself under torch.distributed.run
(one rank per GPU, NCCL); it fails loudly if fewer than N GPUs are visible.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from mch_inputs import CONFIGS, make_medium  # noqa: E402

METRIC = "cell-problem solves/sec per level (L, η, d); HBM GB/s vs B200 ~8 TB/s"
UNIT = "cell-problem solves/s"
HEADLINE = 5


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=HEADLINE)
    ap.add_argument("--impl", default="mch", choices=["mch", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-others", action="store_true", help="skip the per-level lines of the other configs")
    return ap.parse_args()


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def _device_peaks():
    """FP64 FMA and shared-memory peaks measured on this GPU (lib/mch_peaks, DFMA / LDS loops)."""
    exe = os.path.join(ROOT, "paper_2503_01276_b200", "lib", "mch_peaks")
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout.strip().splitlines()[-1]
        return json.loads(out)
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """SM clock + throttle reasons sampled through NVML (pynvml) from a background thread during
    the timed region (every 500 ms: spawning nvidia-smi at 200 ms stalled the driver and
    inflated the step time by ~15%)."""

    def __init__(self, index, period=0.5):
        self.index, self.period, self.rows, self.ok = index, period, [], False

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.hnd = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = nv.nvmlDeviceGetMaxClockInfo(self.hnd, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return
        self.stop_ev = threading.Event()
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.hnd, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.hnd)
                self.rows.append((sm, rs))
            except Exception:
                pass
            self.stop_ev.wait(self.period)

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.stop_ev.set()
        self.thread.join(timeout=5)
        nv = self.nv
        names = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                 "hw_power_brake": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown}
        reasons = sorted({k for _, rs in self.rows for k, bit in names.items() if rs & bit})
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference).  The oracle is test infrastructure; only
# these two legs of bench.py run it.
def _sample_points(cfg):
    """One macropoint per level along the x-axis edge: the corner (0,..,0) at level 1 and
    (η^{L-n}, 0, ..) at level n >= 2 (a chain: each is a child of the previous)."""
    d = cfg.d
    pts = [(0,) * d]
    for lev in range(2, cfg.L + 1):
        pts.append((cfg.eta ** (cfg.L - lev),) + (0,) * (d - 1))
    return pts


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class OracleSample:
    def __init__(self, cfg, kap, ids):
        from oracle import Oracle
        self.cfg = cfg
        self.o = Oracle.from_config(cfg, kap, ids)
        self.pts = _sample_points(cfg)
        self.warm = False

    def step(self):
        """cpu-seconds per macropoint at each level: the sampled points are re-solved with their
        parents' solutions cached (the first call solves the whole ancestry once, untimed)."""
        o = self.o
        if not self.warm:
            for k in self.pts:
                o.solve(k)
            self.warm = True
        per = []
        for k in self.pts:
            o.cache.pop(tuple(k), None)
            t0 = time.process_time()
            o.solve(k)
            per.append(time.process_time() - t0)
        return per

    def value(self, per):
        counts = [len(self.o.plan.S(lev)) for lev in range(1, self.cfg.L + 1)]
        cpu_s = sum(c * p for c, p in zip(counts, per))  # one core
        return sum(counts) * self.cfg.n_rhs / cpu_s

    def text(self):
        return (f"oracle (sparse LU, one core) on one macropoint per level of {self.cfg.name} along the x-axis edge "
                f"{self.pts} with parents cached, cpu-seconds per macropoint x |S_n|; these clipped boundary "
                f"windows are the cheapest of each level, so the rate is an upper bound for the CPU")


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[a.config]
    kap, ids = make_medium(cfg)
    smp = OracleSample(cfg, kap, ids)
    vals = []
    for step in range(a.warmup + a.steps):
        per = smp.step()
        if step >= a.warmup:
            vals.append(smp.value(per))
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_block(cfg, 1),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": smp.text(),
                             "cpu_model": _cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config_block(cfg, world):
    return {"workload": cfg.name, "d": cfg.d, "fine": f"{cfg.n}^{cfg.d}", "H": f"1/{cfg.M}", "L": cfg.L,
            "eta": cfg.eta, "N": cfg.N, "macropoints": (cfg.M + 1) ** cfg.d, "n_rhs": cfg.n_rhs,
            "cell_problems_per_step": (cfg.M + 1) ** cfg.d * cfg.n_rhs,
            "parallelism": f"macropoint-shard x{world}"}


# ------------------------------------------------------------------------------------------
def _flops_per_node_iter(d, level):
    """algorithmic FP64 flops per (level-n node, rhs, PCG iteration): the stencil (2 per
    coefficient: 9-point 2D, 27-point 3D levels >= 2; the 3D level-1 element form, 8 cells x 6)
    plus 14 for the vector updates, dot products and the Jacobi scaling"""
    if d == 2:
        return 2 * 9 + 14
    return (48 if level == 1 else 2 * 27) + 14


def _level_bound(d, level):
    """the 3D level-1/2 windows (22.4 / 4.9 MB of PCG state per macropoint) stream
    through L2/HBM; every 2D level and the 3D levels >= 3 keep the iteration on chip (FP64 / issue
    bound)"""
    return "hbm" if (d == 3 and level <= 2) else "alu"


def _plain_nodes(cfg):
    """Σ over all macropoints of the fine window nodes: the solver DOFs of the plain (L = 1) method
    on the same macropoints, for the cost model"""
    c, n, w2 = cfg.n // cfg.M, cfg.n, 3 * (cfg.n // cfg.M)
    per_dim = []
    for k in range(cfg.M + 1):
        lo = max(0, 2 * k * c - w2) // 2
        hi = min(2 * n, 2 * k * c + w2) // 2
        per_dim.append(hi - lo + 1)
    s = sum(per_dim)
    return s ** cfg.d


def _run_config(cfg, kd, idd, rank, world, steps, warmup, flush, st, barrier, collect=True):
    import torch
    from paper_2503_01276_b200.parallel import ShardedHomogenizer
    sh = ShardedHomogenizer(cfg, kd, idd, rank, world)
    Gd = torch.empty(((cfg.M + 1) ** cfg.d, cfg.n_rhs, cfg.n_rhs), dtype=torch.float64, device="cuda")

    def step():
        sh.reset()
        sh.solve_all()
        sh.effective_coeffs(Gd)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ms, levels = [], []
    for _ in range(steps):
        flush.fill_(1.0)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        step()
        e1.record(st)
        torch.cuda.synchronize()
        barrier()
        ms.append(e0.elapsed_time(e1))
        levels.append([sh.h.level_stats(lev) for lev in range(1, cfg.L + 1)])
    return sh, Gd, ms, levels


def _per_level(cfg, levels, world, peaks_hbm, fp64_tf):
    out = []
    nsteps = len(levels)
    for li in range(cfg.L):
        lev = li + 1
        avg = lambda key: sum(s[li][key] for s in levels) / nsteps  # noqa: E731
        st = levels[-1][li]
        bound = _level_bound(cfg.d, lev)
        pcg_ms = avg("ms_pcg")
        if bound == "hbm":
            ach = avg("pcg_bytes") / (pcg_ms * 1e-3) / 1e9
            frac, unit = ach / peaks_hbm, "GB/s"
        else:
            ach = avg("node_iters") * _flops_per_node_iter(cfg.d, lev) / (pcg_ms * 1e-3) / 1e12
            frac, unit = (ach / fp64_tf if fp64_tf else None), "TFLOP/s"
        out.append({"level": lev, "macropoints": st["macropoints"], "ms": round(avg("ms_total"), 3),
                    "cell_solves_per_s": round(st["problems"] / (avg("ms_total") * 1e-3), 1),
                    "macropoint_solves_per_s": round(st["macropoints"] / (avg("ms_total") * 1e-3), 1),
                    "pcg_ms": round(pcg_ms, 3), "fine_pass_ms": round(avg("ms_setup") + avg("ms_gram"), 3),
                    "comm_ms": round(avg("ms_comm"), 3),
                    "avg_iters": round(st["iters_total"] / max(1, st["problems"]), 1), "max_iters": st["iters_max"],
                    "node_iters": st["node_iters"], "unknowns_level": st["unknowns_level"],
                    "pcg_bound": bound, "pcg_achieved": round(ach, 3), "pcg_unit": unit,
                    "pcg_frac": (round(frac, 4) if frac is not None else None),
                    "rank_deficient": st["rank_deficient"], "launches": st["launches"]})
        tms = avg("ms_transport")
        if lev >= 2 and tms > 0:  # the transport launch (Eqs. 11-13), FP64 / issue bound
            tach = avg("transport_flops") / (tms * 1e-3) / 1e12
            out[-1].update({"transport_ms": round(tms, 3), "transport_units": st["transport_units"],
                            "transport_achieved": round(tach, 3), "transport_unit": "TFLOP/s",
                            "transport_frac": (round(tach / fp64_tf, 4) if fp64_tf else None)})
    return out


def main():
    a = _args()
    if a.impl == "reference":
        return run_reference(a)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.gpus > 1 and "RANK" not in os.environ:
        import torch
        if torch.cuda.device_count() < a.gpus:
            print(json.dumps({"error": f"--gpus {a.gpus} but {torch.cuda.device_count()} GPU(s) visible"}), flush=True)
            sys.exit(2)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000), __file__] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if a.gpus != world:
        print(json.dumps({"error": f"--gpus {a.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev_peaks = _device_peaks() if rank == 0 else {}
    cfg = CONFIGS[a.config]
    kap, ids = make_medium(cfg)
    kd = torch.from_numpy(kap).cuda()
    idd = torch.from_numpy(ids).cuda()
    n_cell = (cfg.M + 1) ** cfg.d * cfg.n_rhs
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2
    st = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    sh, Gd, ms, levels = _run_config(cfg, kd, idd, rank, world, a.steps, a.warmup, flush, st, barrier)
    clk = clocks.stop()
    t = torch.tensor([sum(ms) / len(ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    value = n_cell / (ms_step * 1e-3)
    launches = sum(s["launches"] for s in levels[-1]) + 1  # + the coefficient gather / copy

    pk, pk_src = _peaks()
    fp64_tf = dev_peaks.get("fp64_tflops") if isinstance(dev_peaks, dict) else None
    per_level = _per_level(cfg, levels, world, pk["hbm_gbs"], fp64_tf)
    # dominant kernel: the longest single launch of the step, a level's PCG or its transport
    dom = max(per_level, key=lambda r: r["pcg_ms"])
    domt = max(per_level, key=lambda r: r.get("transport_ms", 0.0))
    lev = dom["level"]
    kname = ("k_pcg2d" if cfg.d == 2 else ("k_pcg3d_l1" if lev == 1 else ("k_pcg3d_w7" if lev == cfg.L and cfg.L >= 4
                                                                          else "k_pcg3d"))) + f" level-{lev} launch"
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r02_dram_per_launch.json")  # ncu --set full, same launch
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(cfg.name, {}).get(f"dram_bytes_pcg_L{lev}_launch")
        except Exception:
            traffic = None
    li = lev - 1
    alg_b = sum(s[li]["pcg_bytes"] for s in levels) / len(levels)
    if dom["pcg_bound"] == "hbm":
        roof = {"kernel": kname, "bound": "hbm", "achieved": dom["pcg_achieved"], "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": dom["pcg_frac"], "traffic": traffic,
                "algorithmic_bytes_per_launch": alg_b, "launch_ms": dom["pcg_ms"], "peak_source": pk_src,
                "algorithmic_bytes": "SURVEY 8(d): 8*(6*nodes*iters per problem + D_n*cells*max_iters per "
                                     "macropoint), D_n = 1 (level 1) / 19 (3D levels >= 2)"}
    else:
        roof = {"kernel": kname, "bound": "alu", "achieved": dom["pcg_achieved"], "peak": fp64_tf, "unit": "TFLOP/s",
                "frac": dom["pcg_frac"], "traffic": traffic, "launch_ms": dom["pcg_ms"],
                "peak_source": "measured FP64 FMA loop (lib/mch_peaks)",
                "algorithmic_flops": "node-iterations x (2 x stencil coefficients + 14)"}
    if domt.get("transport_ms", 0.0) > dom["pcg_ms"]:
        lt = domt["level"]
        ttraffic = None
        if os.path.exists(prof):
            try:
                ttraffic = json.load(open(prof)).get(cfg.name, {}).get(f"dram_bytes_transport_L{lt}_launch")
            except Exception:
                ttraffic = None
        roof = {"kernel": f"k_fine3d_transport level-{lt} launch" if cfg.d == 3 else f"transport level-{lt} launch",
                "bound": "alu", "achieved": domt["transport_achieved"], "peak": fp64_tf, "unit": "TFLOP/s",
                "frac": domt["transport_frac"], "traffic": ttraffic, "launch_ms": domt["transport_ms"],
                "peak_source": "measured FP64 FMA loop (lib/mch_peaks)",
                "algorithmic_flops": "fine window nodes x rhs x (2 npar + 60): I_p from the parents, the "
                                     "kappa-weighted Q1 rows of A_1 I_p, z restriction, constraint sums (DESIGN.md §6)",
                "pcg_dominant": {"kernel": kname, "bound": roof["bound"], "frac": roof["frac"],
                                 "launch_ms": roof["launch_ms"], "traffic": roof["traffic"]}}
    # P10: the paper's cost model: hierarchical solver DOFs / plain-method DOFs
    # vs the model L eta^((1-L) d)
    uk = torch.tensor([float(s["unknowns_level"]) for s in levels[-1]], dtype=torch.float64, device="cuda")
    ni = torch.tensor([float(s["node_iters"]) for s in levels[-1]], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(uk)
        dist.all_reduce(ni)
    plain = _plain_nodes(cfg)
    p10 = {"hier_nodes_per_level": [int(v) for v in uk.tolist()], "plain_nodes": plain,
           "measured_ratio": float(uk.sum().item()) / plain,
           "model_ratio": cfg.L * cfg.eta ** ((1 - cfg.L) * cfg.d),
           "node_iters_per_level": [int(v) for v in ni.tolist()],
           "note": "PAPER.md:488-498: per level (DOFs per local problem) x (macropoints); plain = every "
                   "macropoint on the fine mesh (level 1), model L*eta^((1-L)d)"}

    # e2e through the C ABI with HOST buffers
    kh = torch.from_numpy(kap).pin_memory()
    ih = torch.from_numpy(ids).pin_memory()
    Gh = torch.zeros(((cfg.M + 1) ** cfg.d, cfg.n_rhs, cfg.n_rhs), dtype=torch.float64).pin_memory()
    e2e_ms = []
    for i in range(a.warmup + a.steps):
        flush.fill_(1.0)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sh.set_medium(kh, ih)       # mch_set_medium, host pointers: H2D + device validation
        sh.solve_all()
        sh.effective_coeffs(Gh)     # mch_effective_coeffs into pinned host memory: D2H, synchronises
        e1.record(st)
        torch.cuda.synchronize()
        if i >= a.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
    te = torch.tensor([sum(e2e_ms) / len(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = n_cell / (float(te.item()) * 1e-3)
    sh.close()

    others = {}
    if not a.no_others and world == 1:
        for cid in (2, 3, 4, 5):
            if cid == a.config:
                continue
            c2 = CONFIGS[cid]
            k2, i2 = make_medium(c2)
            sh2, _, ms2, lv2 = _run_config(c2, torch.from_numpy(k2).cuda(), torch.from_numpy(i2).cuda(), rank, world,
                                           2, 1, flush, st, barrier)
            sh2.close()
            m2 = sum(ms2) / len(ms2)
            others[c2.name] = {"ms_per_step": round(m2, 3),
                               "cell_solves_per_s": round((c2.M + 1) ** c2.d * c2.n_rhs / (m2 * 1e-3), 1),
                               "per_level": _per_level(c2, lv2, world, pk["hbm_gbs"], fp64_tf)}

    conf = _config_block(cfg, world)
    conf.update({"l2": "flushed between timed steps (512 MB write)",
                 "macropoint_solves_per_s": (cfg.M + 1) ** cfg.d / (ms_step * 1e-3), "per_level": per_level,
                 "cost_model_P10": p10})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": conf,
        "roofline": roof,
        "device_peaks": dev_peaks,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": kap.nbytes + ids.nbytes,
                "d2h_bytes_per_step": Gh.numel() * 8,
                "path": "mch_set_medium (pinned host kappa/ids) + mch_solve_level 1..L + mch_effective_coeffs "
                        "(pinned host out)"},
        "gpu_launches": launches,
        "clocks": clk,
        "other_configs": others,
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        smp = OracleSample(cfg, kap, ids)
        t0 = time.time()
        smp.step()  # ancestry once
        per = smp.step()
        line["cpu_baseline"] = {"value": smp.value(per), "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": smp.text(), "wall_s": round(time.time() - t0, 1),
                                "cpu_model": _cpu_model()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
