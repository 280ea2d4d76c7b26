import sys, time
sys.path.insert(0, "/root/repo")
import paper_2411_18026_b200 as eb
def run(N, om, reps, lib=None):
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, om)
    mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
    src = eb.AssemblerSource(eb.BlockAssembler(mesh, med, med.default_coupling()))
    tree = eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32))
    for i in range(reps):
        fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
        print(f"N={N} om={om} rep {i}: device {fds.stats().factorize_device_seconds:.4f}s", flush=True)
        del fds
run(262144, 1.0, 2)
run(65536, 4.0, 3)
run(65536, 1.0, 2)
