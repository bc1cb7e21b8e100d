// hpclust/io.hpp: drop-in for the dataset ingest of the reference's io.hpp (io.hpp:17-117):
// delimiter-separated numeric tables to a host Dataset (then uploaded by the device calls) and
// back, with the reference's error types and message texts. The benchmark-campaign result files
// (io.hpp:119-195, over bench.hpp's campaign types) are harness code outside this build.
#pragma once
#include <algorithm>
#include <charconv>
#include <cmath>
#include <fstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <system_error>
#include <vector>

#include "hpclust.hpp"

namespace hpclust {

struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct TableFormat {
    char delimiter = ',';
    bool has_header = false;
};

// Shortest decimal text that reads back as the same double (round trip).
inline std::string format_double(double v) {
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);
    if (r.ec != std::errc{}) throw std::runtime_error("format_double: conversion failed");
    return std::string(buf, r.ptr);
}

// One whole field as a finite double; `where` names the position for the error text.
inline double parse_double(std::string_view field, const std::string& where) {
    double v = 0.0;
    const auto r = std::from_chars(field.data(), field.data() + field.size(), v);
    if (r.ec != std::errc{} || r.ptr != field.data() + field.size())
        throw ParseError("cannot parse numeric field at " + where + ": '" + std::string(field) + "'");
    if (!std::isfinite(v)) throw ParseError("non-finite value at " + where + ": '" + std::string(field) + "'");
    return v;
}

// Rows of `delimiter`-separated reals, all of one width; blank lines are skipped and an optional
// first (header) line is ignored. Row-major into Dataset::values.
inline Dataset load_dataset(const std::string& path, const TableFormat& fmt = {}) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ParseError("cannot open file: " + path);
    Dataset d;
    std::string line;
    std::size_t line_no = 0, width = 0;
    bool skip_header = fmt.has_header;
    while (std::getline(in, line)) {
        ++line_no;
        std::string_view rest(line);
        if (!rest.empty() && rest.back() == '\r') rest.remove_suffix(1);
        if (rest.empty()) continue;
        if (skip_header) {
            skip_header = false;
            continue;
        }
        // field count first (a trailing delimiter makes an empty last field), then the values
        const std::size_t nf = 1 + (std::size_t)std::count(rest.begin(), rest.end(), fmt.delimiter);
        if (width == 0) {
            width = nf;
        } else if (nf != width) {
            throw ParseError("ragged row at line " + std::to_string(line_no) + ": expected " + std::to_string(width) +
                             " fields, got " + std::to_string(nf));
        }
        for (std::size_t col = 1;; ++col) {
            const std::size_t cut = rest.find(fmt.delimiter);
            d.values.push_back(parse_double(rest.substr(0, cut),
                                            "line " + std::to_string(line_no) + ", column " + std::to_string(col)));
            if (cut == std::string_view::npos) break;
            rest.remove_prefix(cut + 1);
        }
        ++d.rows;
    }
    if (d.rows == 0) throw ParseError("no data rows in file: " + path);
    d.cols = width;
    return d;
}

// Ingest to pinned host memory (additive): the parsed values stay in the
// Dataset's own vector, page-locked for the holder's lifetime (hpcg_host_register), so
// DeviceDataset(holder.X) / run(holder.X, cfg) upload at the full PCIe rate. Do not resize
// holder.X.values while it is pinned.
struct PinnedDataset {
    Dataset X;
    bool pinned = false;
    PinnedDataset() = default;
    explicit PinnedDataset(Dataset&& d) : X(std::move(d)) {
        pinned = !X.values.empty() &&
                 hpcg_host_register(X.values.data(), (std::int64_t)(X.values.size() * sizeof(double))) == HPCG_OK;
    }
    PinnedDataset(PinnedDataset&& o) noexcept : X(std::move(o.X)), pinned(o.pinned) { o.pinned = false; }
    PinnedDataset& operator=(PinnedDataset&& o) noexcept {
        release();
        X = std::move(o.X);
        pinned = o.pinned;
        o.pinned = false;
        return *this;
    }
    PinnedDataset(const PinnedDataset&) = delete;
    PinnedDataset& operator=(const PinnedDataset&) = delete;
    ~PinnedDataset() { release(); }

private:
    void release() {
        if (pinned) hpcg_host_unregister(X.values.data());
        pinned = false;
    }
};

inline PinnedDataset load_dataset_pinned(const std::string& path, const TableFormat& fmt = {}) {
    return PinnedDataset(load_dataset(path, fmt));
}

inline void save_dataset(const Dataset& X, const std::string& path, const TableFormat& fmt = {}) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open file for writing: " + path);
    std::string row;
    for (std::size_t i = 0; i < X.rows; ++i) {
        row.clear();
        for (std::size_t c = 0; c < X.cols; ++c) {
            if (c) row.push_back(fmt.delimiter);
            row += format_double(X.values[i * X.cols + c]);
        }
        row.push_back('\n');
        out.write(row.data(), (std::streamsize)row.size());
    }
    if (!out) throw std::runtime_error("write failed: " + path);
}

}  // namespace hpclust
