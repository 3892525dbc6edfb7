"""Multi-GPU sharded query (placeholder; filled in below in this round)."""


def bench_main(args):
    raise NotImplementedError("multi-GPU bench not implemented yet")
