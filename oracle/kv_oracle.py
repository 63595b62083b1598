"""CPU ORACLE (test infrastructure only) — block-hash chain and block keys.

Restates /root/reference/pkg/src/aloraserve/kv_cache.py:
  * hash_block ........... kv_cache.py:41-69 (blake2b-128 via hashlib, the
                           reference's own stdlib dependency)
  * compute_block_keys ... kv_cache.py:72-96 (base-aligned extra keys)
  * chain_digests ........ the fold used by find_cached_prefix / commit_and_free
                           (kv_cache.py:166-182, 253-260)
"""

import hashlib

__all__ = ["DIGEST_SIZE", "DOMAIN", "hash_block", "compute_block_keys", "chain_digests"]

DIGEST_SIZE = 16
DOMAIN = b"aloraserve.block.v1"


def hash_block(parent, tokens, extra_key: str, block_size: int) -> bytes:
    """blake2b-128( DOMAIN | 00 or 01‖parent | u32le(len key) ‖ key | u32le(B) | u32le(tok)×B )."""
    tokens = [int(t) for t in tokens]
    if len(tokens) != block_size:
        raise ValueError(f"block slice has {len(tokens)} tokens, block_size is {block_size}")
    if any(t < 0 or t >= 2**32 for t in tokens):
        raise ValueError("token ids must fit in uint32")
    h = hashlib.blake2b(digest_size=DIGEST_SIZE)
    h.update(DOMAIN)
    if parent is None:
        h.update(b"\x00")
    else:
        if len(parent) != DIGEST_SIZE:
            raise ValueError("parent digest has wrong length")
        h.update(b"\x01" + bytes(parent))
    kb = extra_key.encode()
    h.update(len(kb).to_bytes(4, "little") + kb)
    h.update(len(tokens).to_bytes(4, "little"))
    h.update(b"".join(t.to_bytes(4, "little") for t in tokens))
    return h.digest()


def compute_block_keys(token_seq, block_size, adapter_id=None, inv_start=None) -> list:
    """"" for base blocks; adapter_id for standard LoRA; activated: "" iff (i+1)*B <= inv_start."""
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    n = len(token_seq)
    n_blocks = -(-n // block_size)
    if adapter_id is None:
        if inv_start is not None:
            raise ValueError("inv_start without adapter_id")
        return [""] * n_blocks
    if inv_start is None:
        return [adapter_id] * n_blocks
    if not 0 <= inv_start <= n:
        raise ValueError(f"inv_start {inv_start} outside sequence of length {n}")
    return ["" if (i + 1) * block_size <= inv_start else adapter_id for i in range(n_blocks)]


def chain_digests(tokens, keys, block_size) -> list:
    out, parent = [], None
    for i in range(len(tokens) // block_size):
        parent = hash_block(parent, tokens[i * block_size:(i + 1) * block_size], keys[i], block_size)
        out.append(parent)
    return out
