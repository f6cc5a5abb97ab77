"""Multi-GPU plumbing for SecPE private voting.

Ciphertexts are independent (N/(2n) argmaxes per ciphertext), so a job of
many ciphertexts shards over ranks with no data-path collective: rank r owns a contiguous block of
ciphertexts, every rank derives the same evaluation keys from the client's seed (equivalent to a
one-time broadcast of the public keys), and the only collectives are the timing barrier and the
max-over-ranks reduction of the measured time.  torch.distributed is plumbing only (NCCL on the GPU
box, gloo in the CPU tests).
"""
import torch
import torch.distributed as dist


def shard(n_total, world_size, rank):
    """[begin, end) of the ciphertexts rank `rank` processes (contiguous blocks, sizes differ by <= 1)."""
    if n_total < 0 or world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad shard request")
    base, extra = divmod(n_total, world_size)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def input_seed(config_index, global_ct):
    """Seed of ciphertext `global_ct`'s synthetic scores: a function of its global index only, so the
    sharded job draws exactly the inputs of the single-rank job (no overlap between ranks)."""
    return 1000 * config_index + global_ct


def max_over_ranks(value, device="cpu"):
    """Max of a per-rank float (the job time of a weak-scaling step is the slowest rank's)."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_rank, world_size, ms_max):
    """Whole-job throughput (units/s): all ranks' units over the slowest rank's time."""
    if ms_max <= 0:
        raise ValueError("time must be positive")
    return units_per_rank * world_size / (ms_max / 1000.0)
