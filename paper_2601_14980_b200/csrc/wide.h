// wide.h — program format of the n^2 interpreter kernel (wide.cu), shared with the host (abi.cu).
#pragma once
#include <cstdint>
#include <vector>

namespace pcb {

constexpr int kWideMaxSteps = 160;

enum : uint8_t {
  kSrcReg = 0,       // A: keep the previous result (registers)
  kSrcAcc = 1,       // B: the accumulator slot (squaring)
  kSrcX = 2,         // primary input  #arg of this output (aggregate chunk / single input)
  kSrcB = 3,         // secondary input of this output (hom_add)
  kSrcConst = 4,     // constant #arg (radix limbs, device table)
  kSrcTab = 5,       // per-lane table entry #arg
  kSrcTabDigit = 6,  // table entry = 4-bit digit #arg of this element's scalar (0 -> Montgomery one)
  kSrcOpKeep = 7,    // B: the Op slot as left by the previous step (kPostOp)
  kSrcMatTab = 8,    // matvec power-table entry of (column j, window w), arg = j * 16 + w, digit of E[i][col]
  kSrcGEntry = 9,    // matvec table fill: entry `arg` of this element's own (column, window) table
};
// kPostGTab writes the matvec power-table entry `tab` of window wcur + pad0 of column o; with
// wcur < 0 (fill mode) element o IS the (column, window) pair and the entry is o * 64 + tab.
enum : uint8_t { kPostAcc = 1, kPostTab = 2, kPostOut = 4, kPostOp = 8, kPostGTab = 16 };
constexpr int kMatWin = 6;  // matvec window bits (table of 2^6 powers per column and window)

// constant table layout (ids), per modulus
enum : int { kConstR2 = 0, kConstOneR = 1, kConstOne = 2, kConstFirstF = 3 };

struct WStep {
  uint8_t asrc, aarg, bsrc, barg, post, tab, pad0, pad1;
};

struct MatvecGeom {
  uint32_t* mtab = nullptr;
  const uint64_t* expo = nullptr;
  int cols = 0, nwin = 0, cc = 1, nch = 1, wcur = 0;
  int brows = 0;  // rows per diagonal block (row r uses table columns of block r / brows); 0 = one block
};

struct WideMod {  // host-side constants of one modulus in radix 2^rb
  int rb = 0, n = 0, tpi = 0;
  std::vector<uint32_t> mlimb, mword;
  uint32_t minv = 0;
  int mwords = 0;
};

}  // namespace pcb
