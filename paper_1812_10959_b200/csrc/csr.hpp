// csr.hpp — the host CSR container behind the opaque dic_csr handle
// (synthetic generators and the transaction text parser).
#pragma once

#include <stdint.h>

#include <vector>

struct dic_csr {
    int64_t n = 0;
    std::vector<int64_t> indptr;
    std::vector<int32_t> indices;
};
