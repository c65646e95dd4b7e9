// qsb_internal.hpp — device-side descriptors shared by the host runtime
// (qsb_runtime.cpp) and the sm_100a kernels (qsb_kernels.cu).
//
// A "layer" is one Kronecker product of the reference's fill_layer list
// (unitary_backend.cpp:95-116): identity blocks for untouched qubits and
// instructions, plus the non-identity blocks of the layer's operations.
// Identity blocks never appear explicitly: entry (r, c) of the layer operator
// is zero unless r and c agree on every bit owned by an identity block
// (idmask), and otherwise equals the left-fold product of the non-identity
// block entries in qubit-0-first order — bit-identical to kronecker_fold
// (unitary_backend.cpp:119-125, linalg.cpp:109-129) because a factor of an
// identity block is an exact 1.
#pragma once

#include <cstdint>

namespace qsb {

constexpr int kMaxQubits = 20;  // unitary path: 2 x 16 x 4^n bytes must fit in HBM
constexpr int kMaxBlocks = kMaxQubits;

enum BlockKind : int32_t {
    kBlockGate = 0,        // 2x2 gate_matrix on one qubit            (gates.cpp:40-77)
    kBlockControlled = 1,  // controlled_unitary over a span          (gates.cpp:79-110)
    kBlockTable = 2,       // registered FunctionOp matrix, in HBM    (gates.cpp:127-133)
    kBlockMonomial = 3     // registered matrix with at most one nonzero per row (e.g. the DJ
                           // oracle permutation, circuit_library.cpp:45-58): per row its
                           // column (t_col, -1 if none) and value — the same entries, 2^span
                           // reads instead of 4^span
};

struct BlockDesc {
    int32_t kind;
    int32_t shift;      // n - first - span: bit position of the block's least significant qubit
    int32_t span;       // qubits covered
    uint32_t mask;      // (1 << span) - 1
    uint32_t cmask;     // controlled: control bit within the span (span-1-control_pos)
    uint32_t tmask;     // controlled: target bit within the span
    double u_re[4];     // gate / controlled: 2x2 row-major
    double u_im[4];
    const double* t_re; // table: (2^span)^2 row-major planes; monomial: 2^span row values
    const double* t_im;
    const int32_t* t_col;  // monomial: column of each row's nonzero, or -1
    int32_t mono;          // row -> column map of a monomial block: 0 keep the block's bits
                           // (diagonal), 1 flip the target bit (anti-diagonal u; controlled:
                           // only where the control bit is set), 2 look up t_col
    int32_t pad;
};

struct LayerDesc {
    uint32_t idmask;    // index bits owned by identity blocks
    int32_t nblocks;    // non-identity blocks, qubit-0-first (fold order)
    int32_t real;       // every block entry has an exactly-zero imaginary part
    uint32_t zmask;     // bits on which r and c must agree for a nonzero entry:
                        // identity bits + every controlled block's bits except its target
    int32_t monomial;   // every block is monomial: each operator row has one nonzero
                        // (diagonal / permutation layers: CR, CNOT, X, DJ oracles)
    int32_t pad;
    BlockDesc blocks[kMaxBlocks];
};

// The one-launch paths (K2s: N <= 64; K2m: N = 128, 256) upload and stage this
// compact copy of each layer: the same fields, room for n <= 8 blocks instead of kMaxBlocks.
constexpr int kSmallMaxBlocks = 8;
struct SmallLayerDesc {
    uint32_t idmask;
    int32_t nblocks;
    int32_t real;
    uint32_t zmask;
    int32_t monomial;
    int32_t pad;
    BlockDesc blocks[kSmallMaxBlocks];
};

// Stream-K schedule of the warp-specialised K2: gridDim.x persistent CTAs share
// the T x KT k-tile iterations evenly; a tile split between CTAs is finished by
// the CTA holding its first k-tiles (the "owner"), which adds the partials the
// other CTAs publish in `ws` (flag per tile) in k order — deterministic.
struct SkArgs {
    int enabled = 0;
    int tiles_n = 0;        // output tiles along N
    int tiles = 0;          // T
    int maxc = 0;           // partial slots per tile
    int dp_waves = 0;       // whole-tile data-parallel waves before the stream-K range
    int group_m = 0;        // tile numbering: groups of this many row blocks (0: row-major)
    int zero_skip = 0;      // materialised operand: clear structurally zero B tiles instead of loading them
    double* ws = nullptr;   // [P owner CTAs][maxc][values][256 consumer threads]
    int* flags = nullptr;   // [P owner CTAs], zero between launches (each owner re-arms its own)
    int* dbg = nullptr;     // QSB_SK_DEBUG: protocol anomaly counters
};

// Launch wrappers (qsb_kernels.cu). All return cudaError_t as int.
struct GemmArgs {
    const void* tmap;        // CUtensorMap of the A operand (V, [2][M][N] doubles)
    const LayerDesc* layer;  // host copy, passed by value to the kernel
    double* out;             // [2][M][N]
    int M;
    int N;
    const void* tmap_b = nullptr;  // warp-specialised tiles: CUtensorMap of a materialised
                                   // (transposed) operator; null = generate B in shared memory
    bool real = false;             // 3M warp-specialised tiles: the operator is real -> two real GEMMs
    const void* tmap_real = nullptr;    // two-plane (re, im) view of A for the real variant
    const void* tmap_b_real = nullptr;  // one-plane (re) view of a materialised operator
    SkArgs sk;               // warp-specialised tiles: stream-K schedule (sk.enabled)
    int splits = 1;          // warp-specialised tiles: K split over a thread-block cluster of this
                             // size (1, 2, 4); partial accumulators are summed through
                             // distributed shared memory in rank order (deterministic)
};

// K2c: every GEMM of a chain in one persistent launch (qsb_kernels.cu).
struct ChainArgs {
    const void* tmap3[2];      // 3-plane (re, im, re + im) tensor maps of V buffers 0 / 1
    const void* tmap2[2];      // 2-plane (re, im) views for real layers
    const LayerDesc* layers;   // device array: the operator of GEMM l (l = 0 .. n_gemms - 1)
    int n_gemms;
    double* v[2];              // [3][M][N] each; GEMM l reads v[l & 1], writes v[(l + 1) & 1]
    int M, N;
    int splits;                // k-splits per tile (1, 2, 4, 8)
    double* ws;                // chain_ws_bytes(M, N, splits)
    int* tile_flags;           // [tiles], zeroed by launch_chain
    int* row_done;             // [M / 64], zeroed by launch_chain
};
size_t chain_ws_bytes(int M, int N, int splits);
int launch_chain(const ChainArgs& a, void* stream);

int launch_expand(const LayerDesc& layer, uint32_t row_begin, int M, int N, double* out, int planes,
                  void* stream);
int gemm_tile_planes(int tile);  // planes of the V buffers a tile variant reads/writes (2, or 3 with Vr+Vi)
int launch_zgemm(const GemmArgs& a, int tile, int gemm_mode, void* stream);
// K1t: transposed operator planes for a materialised B (planes 2: re, im; 3: + re+im)
// skip_zero: leave the entries of tiles K2 clears instead of loading (GemmArgs.sk.zero_skip) unwritten
int launch_expand_t(const LayerDesc& layer, int N, double* out, int planes, void* stream, int skip_zero = 0);
int gemm_tile_b_planes(int tile);
// transpose = 1: column blocks (operands L^T, V = U[:, cols]^T). max_free_bits: the
// largest number of free index bits (f) of any layer after the first — 2^f candidate
// entries per operator column, i.e. how much generation work a layer can need.
int launch_small_circuit(const SmallLayerDesc* d_layers, int nlayers, int max_free_bits, int transpose,
                         uint32_t row_begin, int M, int N, const double* x, double* v, double* psi, void* stream);
// rows [col_begin, col_begin + M) of L^T (the first layer of a column block)
int launch_expand_cols(const LayerDesc& layer, uint32_t col_begin, int M, int N, double* out, int planes,
                       void* stream);
// psi[k] = sum_{i in [i0, i0 + count)} V[i][k] x[col0 + i - i0] (column blocks; psi has N entries)
int launch_matvec_t(const double* v, int M, int N, int i0, int count, int col0, const double* x, double* psi,
                    void* stream);
int launch_matvec(const double* v, int M, int N, const double* x, double* psi, void* stream);
int launch_probabilities(const double* psi, int64_t dim, double* p, double* partial, int partial_cap,
                         double* norm, void* stream);

// Registry validation (qsb_registry.cu): is_unitary via a DMMA Gram matrix.
int registry_configure();
int gram_tile();
int launch_transpose(const double* re, const double* im, double* t, int N, void* stream);
int launch_gram(const void* tmapT, int N, unsigned long long* maxdev, void* stream);
int launch_gram_small(const double* re, const double* im, int N, unsigned long long* maxdev, void* stream);

// Tile shapes of the K2 GEMM (rows x cols of the output tile).
enum GemmTile : int { kTile128x64 = 0, kTile64x64 = 1, kTile32x32 = 2, kTileWs4M = 3, kTileWs3M = 4, kTileWs3MS = 5 };
int configure_kernels();
int ws_max_active_clusters(int splits);  // co-resident clusters of the warp-specialised K2 per split size
int ws_partial_values(int tile);          // accumulator values per consumer thread of a tile variant
int gemm_tile_rows(int tile);
int gemm_tile_cols(int tile);
size_t small_circuit_smem_bytes(int M, int N);
int mid_three_m();  // K2m computes complex layers as 3M (1) or 4M (0)

}  // namespace qsb
