"""Lab: swarm_adapter.validate_files sharded over N NCCL ranks with the GPU backend, compared
with the single-process verdicts on the same corpus (honest files, every Forge attack class,
tampered proofs).  Rank 0 prints one JSON line.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \\
        tools/lab/validate_files_dist.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import torch.distributed as dist

    from refpath import add_ref_to_path
    add_ref_to_path()
    import test_swarm_adapter as T
    from paper_2505_07291_b200 import swarm_adapter
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    forge, ctx = T.fixtures()
    ctx.commit_q = 0.5
    swarm_adapter.install("toploc", backend=swarm_adapter.GpuBackend())  # the Forge then writes TOPLOC proofs
    blobs = T.corpus(forge)
    got = swarm_adapter.validate_files(blobs, ctx)            # sharded over the ranks
    dist.barrier()
    if rank == 0:
        dist.destroy_process_group()
        single = swarm_adapter.validate_files(blobs, ctx)      # this process alone
        key = lambda vs: [(v.result, v.failed_check, v.details) for v in vs]
        print(json.dumps({"ranks": int(os.environ["WORLD_SIZE"]), "files": len(blobs),
                          "equal_to_single_process": key(got) == key(single),
                          "accepted": sum(v.result == "accept" for v in got),
                          "checks": sorted({v.failed_check for v in got if v.failed_check})}))
    else:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
