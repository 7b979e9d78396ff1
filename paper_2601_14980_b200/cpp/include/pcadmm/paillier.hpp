// Drop-in include path for code written against the reference (#include "pcadmm/paillier.hpp"):
// the B200 facade.  Build with -I paper_2601_14980_b200/cpp/include, link libpcadmm_b200.so.
#pragma once
#include "../../pcb200_pcadmm.hpp"
