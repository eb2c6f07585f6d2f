// geoshoot/pipeline.hpp -- point-cloud files and rigid pre-alignment on
// either side of the hot path (reference pipeline.hpp:11-68): xyz text and
// legacy-VTK ASCII polydata (gs_read_points / gs_write_points), and the
// least-squares rigid Procrustes alignment (gs_procrustes_align).
#pragma once

#include <array>
#include <string>
#include <vector>

#include "geoshoot/core.hpp"

namespace geoshoot {

struct RigidTransform {
  std::array<Vec3, 3> rotation_rows;  // orthonormal, det = +1
  Vec3 translation;
  Vec3 apply(const Vec3& x) const {
    return {dot(rotation_rows[0], x) + translation.x, dot(rotation_rows[1], x) + translation.y,
            dot(rotation_rows[2], x) + translation.z};
  }
  static RigidTransform identity() { return {{Vec3{1, 0, 0}, Vec3{0, 1, 0}, Vec3{0, 0, 1}}, Vec3{}}; }
};

struct ProcrustesResult {
  RigidTransform transform;
  PointSet aligned;
};

/// Rotation + translation (no scaling) taking source onto target under index
/// correspondence, reflection-corrected; N >= 3 non-collinear points.
ProcrustesResult procrustes_align(const PointSet& source, const PointSet& target);

enum class PointFormat { XyzText, LegacyPolydataAscii };

PointFormat format_for_path(const std::string& path);
PointSet read_points(const std::string& path, PointFormat format);
void write_points(const PointSet& points, const std::string& path, PointFormat format,
                  const std::vector<std::string>& header_comments = {});

}  // namespace geoshoot
