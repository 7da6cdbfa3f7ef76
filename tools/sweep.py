"""Device timing sweep over configs / partition counts (dev tool)."""
import sys, time
import torch
sys.path.insert(0, "/root/repo")
import btagen
import paper_2503_17528_b200 as sb

CFG = {"C2": (128, 1024, 64), "C3": (365, 2048, 4), "C4": (256, 512, 16), "C5": (16384, 64, 8)}


def flops(n, b, a):
    F = (n - 1) * (7 / 3 * b**3 + 3 * a * b * b + a * a * b) + b**3 / 3 + a * b * b + a * a * b + a**3 / 3
    S = (n - 1) * (14 / 3 * b**3 + 6 * a * b * b + 2 * a * a * b) + 2 * b**3 / 3 + 2 * a * b * b + 2 * a * a * b + 2 * a**3 / 3
    return F + S


def run(name, Ps, reps=2):
    n, b, a = CFG[name]
    A0 = btagen.g1_torch(0, n, b, a)
    D = {k: v.clone() for k, v in A0.items()}
    fl = flops(n, b, a)
    for P in Ps:
        try:
            t0 = time.time()
            if P == "auto":
                P = sb.auto_partitions(n, b)
            if P == 1 or P == [1]:
                P = 1
                sb.graph_stats(2, n, b, a)
            elif isinstance(P, int):
                sb.graph_stats(3, n, b, a, P)
            tb = time.time() - t0
            best = 1e9
            for r in range(reps):
                for k in D:
                    D[k].copy_(A0[k])
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                if P == 1:
                    ld = sb.selinv(D["diag"], D["lower"], D["arrow"], D["tip"], check=False)
                else:
                    ld = sb.pselinv(D["diag"], D["lower"], D["arrow"], D["tip"], P, check=False)
                e1.record(); torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            info = int(sb.default_handle().scalars()[0].item())
            print(f"{name} n={n} b={b} a={a} P={P}: {best:.2f} ms  {fl / best / 1e9:.2f} TFLOP/s  (build {tb:.1f}s, info {info})", flush=True)
        except Exception as e:
            print(f"{name} P={P}: error {e}", flush=True)
    del A0, D
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        name, ps = spec.split(":")
        run(name, [x if x == "auto" else ([int(y) for y in x.split("x")] if "x" in x else int(x))
                   for x in ps.split(",")])
