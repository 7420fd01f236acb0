// TEST BUILD ONLY: plain types shared by the two engine sides.
#pragma once
#include <cstddef>
#include <string>
#include <vector>

struct SideStatement {
    std::string tag, error;
    std::vector<std::vector<std::string>> rows;
    std::vector<std::string> notices;
    std::size_t batches = 0;
};

struct SideResult {
    std::vector<SideStatement> statements;
    std::size_t cache_builds = 0, cache_hits = 0, cache_adopted = 0;
};

std::string engine_ref_load(const std::string& csv);
std::string engine_dev_load(const std::string& csv);

SideResult engine_ref(const std::string& csv, const std::vector<std::string>& sqls);
SideResult engine_dev(const std::string& csv, const std::vector<std::string>& sqls);
