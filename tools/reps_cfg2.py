import sys, time
sys.path.insert(0, '/root/repo')
import paper_2002_03400_b200 as B
w = B.configs.build(2)
for r in range(12):
    t = time.perf_counter()
    bf, log = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    slow = max(log.phases, key=lambda p: p.seconds)
    print(f"rep {r}: {log.total_seconds:.4f} s wall {time.perf_counter()-t:.4f} peak_probes {log.peak_concurrent_probes} slowest {slow.name} {slow.seconds*1e3:.1f} ms", flush=True)
