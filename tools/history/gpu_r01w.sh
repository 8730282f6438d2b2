./tools/ubench/pool 0; echo ---; ./tools/ubench/pool 1
