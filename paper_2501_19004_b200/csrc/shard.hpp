// Device side of the row-sharded engine (shard.cu).
#pragma once

#include "kernels.cuh"

namespace lvn {

// local offsets of the own rows [v0, v1) of a global CSR: out[u] =
// clamp(off[u], off[v0], off[v1]) - off[v0] for u in [0, n] (other rows empty)
void shard_offsets(const u64* off, u32 n, u32 v0, u32 v1, u64* out, cudaStream_t s);
// bits of one community id in a packed (row, target) key
u32 key_bits(u32 count);
// partial super-edges of the own rows: (C[u] << kb | C[v], sum of w in fp64),
// sorted by key, distinct keys at the front of keys / vals; returns their number
u64 partial_super_edges(const DGraph& g, const u32* C, u32 v0, u32 v1, u32 kb, DBuf<ull>& keys, DBuf<double>& vals,
                        cudaStream_t s);
// holey partial super-rows (aggregate_device with PartialRows) flattened to
// (row << kb | target, fp64 w) entries in row order; returns their number
u64 holey_entries(const u64* hoff, const u32* htgt, const double* hw64, const u32* fill, u32 count, u32 kb,
                  DBuf<ull>& keys, DBuf<double>& vals, cudaStream_t s);
// cnt[c] = entries of row c among n sorted keys (cnt zeroed here, count entries)
void super_row_counts(const ull* keys, u64 n, u32 count, u32 kb, u32* cnt, cudaStream_t s);
// cut[k] = first entry whose row reaches cb[k] (k < parts), cut[parts] = n
void route_entries(const ull* keys, u64 n, const u32* cb, int parts, u32 kb, u64* cut, cudaStream_t s);
// received entries -> this rank's super-rows (over all `count` rows, the
// others empty): stable sort, fp64 sum per key, one f32 narrowing; *tw gets
// the summed f32 weights (fp64, device)
void merge_super_rows(DBuf<ull>& keys, DBuf<double>& vals, u64 n, u32 count, u32 kb, OwnedCsr& out, double* tw,
                      cudaStream_t s);
// len[u] = off[u+1] - off[u] (u32), u < n
void row_lengths(const u64* off, u32 n, u32* len, cudaStream_t s);
// flags[u] = 0 outside [v0, v1)
void zero_outside(u8* flags, u32 n, u32 v0, u32 v1, cudaStream_t s);

}  // namespace lvn
